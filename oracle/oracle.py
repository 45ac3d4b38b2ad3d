"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end for the two CPU checkers.

* ``Oracle``    — the C restatement in ``oracle/sparsek_oracle.c`` (always built
  by ``make -C oracle``; travels to the GPU box as ``oracle/_build/liboracle.so``).
* ``Reference`` — the unmodified reference compiled from /root/reference by the
  same Makefile into ``oracle/_ref/libsparsek_ref.so`` (git-ignored; shipped to
  the GPU box with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module. The product path (``paper_2406_16747_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsek_ref.so")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i32(a):
    return a.ctypes.data_as(_i32p) if a is not None else None


def _i64(a):
    return a.ctypes.data_as(_i64p) if a is not None else None


def build():
    """Compile the checkers (the reference only where its sources exist)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class OracleError(RuntimeError):
    pass


class _OrcCfg(C.Structure):
    _fields_ = [("k", C.c_double), ("window", C.c_int64), ("heads", C.c_int64),
                ("scale", C.c_double), ("key_soft", C.c_int32), ("mask_st", C.c_int32)]


@dataclass
class Selection:
    tau_q: np.ndarray      # [L] tau each query froze (-inf when unbound)
    n_sel: np.ndarray      # [L] int32
    att_off: np.ndarray    # [L+1] int64
    att: np.ndarray        # [total] int32 (selected asc, then window asc, then self)
    gate: np.ndarray       # [total] aligned with att (1.0 on non-selected entries)

    def sel_of(self, i):
        b = self.att_off[i]
        return self.att[b:b + self.n_sel[i]]

    def att_of(self, i):
        return self.att[self.att_off[i]:self.att_off[i + 1]]


class Oracle:
    """The C restatement (sparsek_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)

    def _rc(self, rc, what):
        if rc != 0:
            raise OracleError(f"{what}: oracle error code {rc}")

    # scoring ------------------------------------------------------------
    def score_fwd(self, x, w, norm_mode=1, slope_order=1, slope_enabled=True, slope_eps=0.01):
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        L, D = x.shape
        raw, u, mean, sdev = (np.zeros(L) for _ in range(4))
        self._rc(self.lib.orc_score_fwd(_d(x), _d(w), C.c_int64(L), C.c_int64(D),
                                        C.c_int32(norm_mode), C.c_int32(slope_order),
                                        C.c_int32(int(slope_enabled)), C.c_double(slope_eps),
                                        _d(raw), _d(u), _d(mean), _d(sdev)), "score_fwd")
        return raw, u, mean, sdev

    def score_bwd(self, gu, raw, mean, sdev, norm_mode=1):
        gu, raw, mean, sdev = (np.ascontiguousarray(a, np.float64) for a in (gu, raw, mean, sdev))
        graw = np.zeros_like(gu)
        self.lib.orc_score_bwd(_d(gu), _d(raw), _d(mean), _d(sdev), C.c_int64(len(gu)),
                               C.c_int32(norm_mode), _d(graw))
        return graw

    # operator -----------------------------------------------------------
    def sparsek(self, z, k):
        z = np.ascontiguousarray(z, np.float64)
        p = np.zeros_like(z)
        tau = C.c_double()
        uc, wc = C.c_int64(), C.c_int64()
        deg, inf = C.c_int32(), C.c_int32()
        self._rc(self.lib.orc_sparsek(_d(z), C.c_int64(len(z)), C.c_double(k), _d(p),
                                      C.byref(tau), C.byref(uc), C.byref(wc), C.byref(deg),
                                      C.byref(inf)), "sparsek")
        return dict(p=p, tau=tau.value, u_count=uc.value, w_count=wc.value,
                    degenerate=bool(deg.value), infeasible=bool(inf.value))

    def sparsek_jvp(self, z, k, v):
        z = np.ascontiguousarray(z, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(z)
        self._rc(self.lib.orc_sparsek_jvp(_d(z), C.c_int64(len(z)), C.c_double(k), _d(v),
                                          _d(out)), "sparsek_jvp")
        return out

    def topk_hard(self, z, k):
        z = np.ascontiguousarray(z, np.float64)
        out = np.zeros_like(z)
        self.lib.orc_topk_hard(_d(z), C.c_int64(len(z)), C.c_int64(k), _d(out))
        return out

    def stream_taus(self, z, k):
        z = np.ascontiguousarray(z, np.float64)
        tau = np.zeros_like(z)
        ins = np.zeros(len(z), np.uint8)
        self._rc(self.lib.orc_stream_taus(_d(z), C.c_int64(len(z)), C.c_double(k), _d(tau),
                                          ins.ctypes.data_as(_u8p)), "stream")
        return tau, ins.astype(bool)

    # retention / attention ---------------------------------------------
    def select(self, u, k, window) -> Selection:
        u = np.ascontiguousarray(u, np.float64)
        L = len(u)
        tau_q = np.zeros(L)
        n_sel = np.zeros(L, np.int32)
        att_off = np.zeros(L + 1, np.int64)
        self._rc(self.lib.orc_select(_d(u), C.c_int64(L), C.c_double(k), C.c_int64(window),
                                     _d(tau_q), _i32(n_sel), _i64(att_off), None, None), "select")
        total = int(att_off[L])
        att = np.zeros(max(total, 1), np.int32)
        gate = np.zeros(max(total, 1))
        self._rc(self.lib.orc_select(_d(u), C.c_int64(L), C.c_double(k), C.c_int64(window),
                                     _d(tau_q), _i32(n_sel), _i64(att_off), _i32(att), _d(gate)),
                 "select")
        return Selection(tau_q, n_sel, att_off, att[:total], gate[:total])

    def _cfg(self, k, window, heads, scale=0.0, key_mode="hard", mask_mode="soft"):
        return _OrcCfg(float(k), int(window), int(heads), float(scale),
                       int(key_mode == "soft"), int(mask_mode == "straight_through"))

    def attn_fwd(self, q, k, v, sel: Selection, *, kbudget, window, scale=0.0, key_mode="hard",
                 mask_mode="soft"):
        """q/k/v: [L, H, p] float64. Returns (o [L,H,p], maxa [L,H], denom [L,H])."""
        q, k, v = (np.ascontiguousarray(a, np.float64) for a in (q, k, v))
        L, H, p = q.shape
        cfg = self._cfg(kbudget, window, H, scale, key_mode, mask_mode)
        o = np.zeros_like(q)
        maxa = np.zeros((L, H))
        den = np.zeros((L, H))
        self._rc(self.lib.orc_attn_fwd(_d(q), _d(k), _d(v), C.c_int64(L), C.c_int64(p),
                                       C.byref(cfg), _i32(sel.n_sel), _i64(sel.att_off),
                                       _i32(sel.att), _d(sel.gate), _d(o), _d(maxa), _d(den)),
                 "attn_fwd")
        return o, maxa, den

    def attn_bwd(self, q, k, v, do, u, sel: Selection, maxa, denom, *, kbudget, window, scale=0.0,
                 key_mode="hard", mask_mode="soft"):
        """Returns (dq, dk, dv [L,H,p], gu [L])."""
        q, k, v, do = (np.ascontiguousarray(a, np.float64) for a in (q, k, v, do))
        u = np.ascontiguousarray(u, np.float64)
        maxa = np.ascontiguousarray(maxa, np.float64)
        denom = np.ascontiguousarray(denom, np.float64)
        L, H, p = q.shape
        cfg = self._cfg(kbudget, window, H, scale, key_mode, mask_mode)
        dq, dk, dv = (np.zeros_like(q) for _ in range(3))
        gu = np.zeros(L)
        self._rc(self.lib.orc_attn_bwd(_d(q), _d(k), _d(v), _d(do), C.c_int64(L), C.c_int64(p),
                                       C.byref(cfg), _d(u), _d(sel.tau_q), _i32(sel.n_sel),
                                       _i64(sel.att_off), _i32(sel.att), _d(sel.gate), _d(maxa),
                                       _d(denom), _d(dq), _d(dk), _d(dv), _d(gu)), "attn_bwd")
        return dq, dk, dv, gu


# ---------------------------------------------------------------------------
# The compiled reference (oracle/_ref/libsparsek_ref.so).


class _RefCfg(C.Structure):
    _fields_ = [("k", C.c_double), ("window", C.c_uint64), ("heads", C.c_uint64),
                ("scale", C.c_double), ("key_mode", C.c_int32), ("mask_mode", C.c_int32),
                ("group_size", C.c_uint64), ("slope_eps", C.c_double),
                ("slope_enabled", C.c_int32), ("norm_mode", C.c_int32),
                ("slope_order", C.c_int32), ("pad_", C.c_int32)]


def ref_cfg(k, window, heads=1, scale=0.0, key_mode="hard", mask_mode="soft", group_size=128,
            slope_eps=0.01, slope_enabled=True, norm_mode="timestep_norm",
            slope_order="norm_then_slope"):
    return _RefCfg(float(k), int(window), int(heads), float(scale), int(key_mode == "soft"),
                   int(mask_mode == "straight_through"), int(group_size), float(slope_eps),
                   int(bool(slope_enabled)), int(norm_mode == "timestep_norm"),
                   int(slope_order == "norm_then_slope"), 0)


class ReferenceError_(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class RefTape:
    y: np.ndarray
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    head_concat: np.ndarray
    raw: np.ndarray
    u: np.ndarray
    norm_mean: np.ndarray
    norm_sdev: np.ndarray
    tau_push: np.ndarray
    n_sel: np.ndarray
    att_off: np.ndarray
    att: np.ndarray
    gate: np.ndarray     # selected entries only (reference layout)
    maxa: np.ndarray     # [L, H]
    denom: np.ndarray    # [L, H]


class Reference:
    """The reference library itself, compiled from /root/reference."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _rc(self, rc):
        if rc != 0:
            raise ReferenceError_(rc, self.lib.ref_last_error().decode())

    def sparsek(self, z, k, sort_cap=0):
        z = np.ascontiguousarray(z, np.float64)
        p = np.zeros_like(z)
        tau = C.c_double()
        uc, wc = C.c_uint64(), C.c_uint64()
        deg, inf = C.c_int32(), C.c_int32()
        self._rc(self.lib.ref_sparsek(_d(z), C.c_uint64(len(z)), C.c_double(k),
                                      C.c_uint64(sort_cap), _d(p), C.byref(tau), C.byref(uc),
                                      C.byref(wc), C.byref(deg), C.byref(inf)))
        return dict(p=p, tau=tau.value, u_count=uc.value, w_count=wc.value,
                    degenerate=bool(deg.value), infeasible=bool(inf.value))

    def sparsek_jvp(self, z, k, v):
        z = np.ascontiguousarray(z, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(z)
        self._rc(self.lib.ref_sparsek_jvp(_d(z), C.c_uint64(len(z)), C.c_double(k), _d(v),
                                          _d(out)))
        return out

    def topk_hard(self, z, k):
        z = np.ascontiguousarray(z, np.float64)
        out = np.zeros_like(z)
        self._rc(self.lib.ref_topk_hard(_d(z), C.c_uint64(len(z)), C.c_uint64(k), _d(out)))
        return out

    def stream(self, z, k, heap_cap=0):
        z = np.ascontiguousarray(z, np.float64)
        n = len(z)
        tau = np.zeros(n)
        ins = np.zeros(n, np.uint8)
        surv = np.zeros(n, np.uint64)
        p_last = np.zeros(n)
        self._rc(self.lib.ref_stream_run(_d(z), C.c_uint64(n), C.c_double(k),
                                         C.c_uint64(heap_cap), _d(tau), ins.ctypes.data_as(_u8p),
                                         surv.ctypes.data_as(C.POINTER(C.c_uint64)), _d(p_last)))
        return tau, ins.astype(bool), surv.astype(np.int64), p_last

    def stream_blob(self, z, k, heap_cap=0):
        """StreamState::serialize after pushing z (proj/src/stream.cpp:224-252)."""
        z = np.ascontiguousarray(z, np.float64)
        used = C.c_uint64()
        self._rc(self.lib.ref_stream_blob(_d(z), C.c_uint64(len(z)), C.c_double(k),
                                          C.c_uint64(heap_cap), None, C.c_uint64(0), C.byref(used)))
        buf = (C.c_uint8 * used.value)()
        self._rc(self.lib.ref_stream_blob(_d(z), C.c_uint64(len(z)), C.c_double(k),
                                          C.c_uint64(heap_cap), buf, C.c_uint64(used.value),
                                          C.byref(used)))
        return bytes(buf)

    def stream_resume(self, blob, z):
        """StreamState::deserialize(blob), push z; per-push tau."""
        z = np.ascontiguousarray(z, np.float64)
        tau = np.zeros(len(z))
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self._rc(self.lib.ref_stream_resume(buf, C.c_uint64(len(blob)), _d(z), C.c_uint64(len(z)),
                                            _d(tau)))
        return tau

    def attention(self, x, wq, wk, wv, wo, w_score, cfg, use_float=False, grad_out=None,
                  chunk_len=0):
        """Forward with tape (+ backward when grad_out is given); chunk_len > 0
        runs the reference's chunked_forward (Algorithm 3)."""
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        w_score = np.ascontiguousarray(w_score, np.float64)
        L, D = x.shape
        h = C.c_void_p()
        self._rc(self.lib.ref_attention_fwd_chunked(C.c_int32(int(use_float)), C.c_uint64(L),
                                                    C.c_uint64(D), _d(x), _d(wq), _d(wk), _d(wv),
                                                    _d(wo), _d(w_score), C.byref(cfg),
                                                    C.c_uint64(int(chunk_len)), C.byref(h)))
        try:
            n, ta, ts, nt = (C.c_uint64() for _ in range(4))
            self._rc(self.lib.ref_tape_sizes(h, C.byref(n), C.byref(ta), C.byref(ts),
                                              C.byref(nt)))
            H = int(cfg.heads)
            arr = lambda *s: np.zeros(s)
            y, q, k, v, hc = (arr(L, D) for _ in range(5))
            raw, u, nm, ns = (arr(L) for _ in range(4))
            tau = arr(max(int(nt.value), 1))
            n_sel = np.zeros(L, np.uint32)
            att_off = np.zeros(L + 1, np.uint64)
            att = np.zeros(max(int(ta.value), 1), np.uint32)
            gate = arr(max(int(ts.value), 1))
            maxa, den = arr(L, H), arr(L, H)
            self._rc(self.lib.ref_tape_copy(
                h, _d(y), _d(q), _d(k), _d(v), _d(hc), _d(raw), _d(u), _d(nm), _d(ns), _d(tau),
                n_sel.ctypes.data_as(C.POINTER(C.c_uint32)),
                att_off.ctypes.data_as(C.POINTER(C.c_uint64)),
                att.ctypes.data_as(C.POINTER(C.c_uint32)), _d(gate), _d(maxa), _d(den)))
            tape = RefTape(y, q, k, v, hc, raw, u, nm, ns, tau[:int(nt.value)],
                           n_sel.astype(np.int32), att_off.astype(np.int64),
                           att[:int(ta.value)].astype(np.int32), gate[:int(ts.value)], maxa, den)
            grads = None
            if grad_out is not None:
                g = np.ascontiguousarray(grad_out, np.float64)
                dx = arr(L, D)
                dwq, dwk, dwv, dwo = (arr(D, D) for _ in range(4))
                dws = arr(D)
                self._rc(self.lib.ref_tape_backward(h, _d(g), _d(dx), _d(dwq), _d(dwk), _d(dwv),
                                                    _d(dwo), _d(dws)))
                grads = dict(dx=dx, dwq=dwq, dwk=dwk, dwv=dwv, dwo=dwo, dw_score=dws)
            return tape, grads
        finally:
            self.lib.ref_tape_free(h)

    def stream_events(self, z, k, heap_cap=0):
        """Per push: (tau, inserted, cap_forced, evicted list) from StreamStepResult."""
        z = np.ascontiguousarray(z, np.float64)
        n = len(z)
        tau = np.zeros(n)
        ins, capf = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        cnt = np.zeros(n, np.uint64)
        flat = np.zeros(max(n, 1), np.uint64)
        u64p = C.POINTER(C.c_uint64)
        self._rc(self.lib.ref_stream_events(_d(z), C.c_uint64(n), C.c_double(k), C.c_uint64(heap_cap),
                                            _d(tau), ins.ctypes.data_as(_u8p), capf.ctypes.data_as(_u8p),
                                            cnt.ctypes.data_as(u64p), flat.ctypes.data_as(u64p),
                                            C.c_uint64(len(flat))))
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        evs = [flat[off[t]:off[t + 1]].astype(np.int64).tolist() for t in range(n)]
        return tau, ins.astype(bool), capf.astype(bool), evs

    def stream_mask(self, z, k, heap_cap=0):
        """stream_mask after pushing z: (positions, hard, soft, indices)."""
        z = np.ascontiguousarray(z, np.float64)
        n = len(z)
        pos, idx = np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.uint64)
        hard, soft = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        nn, ni = C.c_uint64(), C.c_uint64()
        u64p = C.POINTER(C.c_uint64)
        self._rc(self.lib.ref_stream_mask(_d(z), C.c_uint64(n), C.c_double(k), C.c_uint64(heap_cap),
                                          pos.ctypes.data_as(u64p), _d(hard), _d(soft), C.byref(nn),
                                          idx.ctypes.data_as(u64p), C.byref(ni)))
        m = nn.value
        return (pos[:m].astype(np.int64), hard[:m], soft[:m], idx[:ni.value].astype(np.int64))

    def sparsek_st(self, z, k):
        z = np.ascontiguousarray(z, np.float64)
        fwd, p = np.zeros_like(z), np.zeros_like(z)
        self._rc(self.lib.ref_sparsek_st(_d(z), C.c_uint64(len(z)), C.c_double(k), _d(fwd), _d(p)))
        return fwd, p

    def sparsek_partial_stats(self, z, k, sort_cap):
        z = np.ascontiguousarray(z, np.float64)
        p = np.zeros_like(z)
        tau = C.c_double()
        calls, fb = C.c_uint64(), C.c_uint64()
        self._rc(self.lib.ref_sparsek_partial_stats(_d(z), C.c_uint64(len(z)), C.c_double(k),
                                                    C.c_uint64(sort_cap), _d(p), C.byref(tau),
                                                    C.byref(calls), C.byref(fb)))
        return p, tau.value, calls.value, fb.value

    def dense_attention_grads(self, x, wq, wk, wv, wo, grad_out, heads=1):
        """dense_causal_attention + dense_causal_attention_backward (double)."""
        x, wq, wk, wv, wo, g = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo, grad_out))
        L, D = x.shape
        y, dx = np.zeros((L, D)), np.zeros((L, D))
        dws = [np.zeros((D, D)) for _ in range(4)]
        self._rc(self.lib.ref_dense_attention_grads(C.c_uint64(L), C.c_uint64(D), C.c_uint64(heads), _d(x),
                                                    _d(wq), _d(wk), _d(wv), _d(wo), _d(g), _d(y), _d(dx),
                                                    *[_d(a) for a in dws]))
        return y, dict(dx=dx, dwq=dws[0], dwk=dws[1], dwv=dws[2], dwo=dws[3])

    def dense_attention(self, x, wq, wk, wv, wo, heads=1):
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        L, D = x.shape
        y = np.zeros((L, D))
        self._rc(self.lib.ref_dense_attention(C.c_uint64(L), C.c_uint64(D), C.c_uint64(heads),
                                              _d(x), _d(wq), _d(wk), _d(wv), _d(wo), _d(y)))
        return y

    def decode(self, x, wq, wk, wv, wo, w_score, cfg, prompt, use_float=False):
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        w_score = np.ascontiguousarray(w_score, np.float64)
        L, D = x.shape
        y = np.zeros((L, D))
        peak = C.c_uint64()
        self._rc(self.lib.ref_decode_run(C.c_int32(int(use_float)), C.c_uint64(L), C.c_uint64(D),
                                         C.c_uint64(prompt), _d(x), _d(wq), _d(wk), _d(wv),
                                         _d(wo), _d(w_score), C.byref(cfg), _d(y),
                                         C.byref(peak)))
        return y, int(peak.value)

    def cache_blob(self, x, wq, wk, wv, wo, w_score, cfg, prompt, use_float=False):
        """Run rows of x (forward_chunk on the prompt, generate_step after) and
        return (y, SparseKvCache::serialize payload)."""
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        w_score = np.ascontiguousarray(w_score, np.float64)
        n, D = x.shape
        y = np.zeros((n, D))
        used = C.c_uint64()
        args = lambda buf, cap: (C.c_int32(int(use_float)), C.c_uint64(n), C.c_uint64(D), C.c_uint64(prompt),
                                 _d(x), _d(wq), _d(wk), _d(wv), _d(wo), _d(w_score), C.byref(cfg), _d(y),
                                 buf, C.c_uint64(cap), C.byref(used))
        self._rc(self.lib.ref_cache_blob(*args(None, 0)))
        buf = (C.c_uint8 * used.value)()
        self._rc(self.lib.ref_cache_blob(*args(buf, used.value)))
        return y, bytes(buf)

    def cache_resume(self, blob, x, wq, wk, wv, wo, w_score, cfg, use_float=False):
        """SparseKvCache::deserialize(blob) then generate_step over the rows of x."""
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        w_score = np.ascontiguousarray(w_score, np.float64)
        n, D = x.shape
        y = np.zeros((n, D))
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self._rc(self.lib.ref_cache_resume(C.c_int32(int(use_float)), buf, C.c_uint64(len(blob)),
                                           C.c_uint64(n), C.c_uint64(D), _d(x), _d(wq), _d(wk), _d(wv),
                                           _d(wo), _d(w_score), C.byref(cfg), _d(y)))
        return y

    def bench_units(self, units, threads, L, p, k, window, seed=1, with_bwd=True):
        secs = C.c_double()
        self._rc(self.lib.ref_bench_units(C.c_uint64(units), C.c_uint64(threads), C.c_uint64(L),
                                          C.c_uint64(p), C.c_double(k), C.c_uint64(window),
                                          C.c_uint64(seed), C.c_int32(int(with_bwd)),
                                          C.byref(secs)))
        return secs.value


    def linear_mix(self, x, wq, wk, wv, wo, w_score, feat, cfg, use_float=False, grad_out=None,
                   chunk_len=0):
        """linear_mix_attention (+ its backward when grad_out is given):
        (y, {dx, dwq, dwk, dwv, dwo, dw_score, dfeat} or None)."""
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        L, D = x.shape
        ws = np.ascontiguousarray(w_score if w_score is not None else np.zeros(D), np.float64)
        f = np.ascontiguousarray(feat, np.float64)
        y = np.zeros((L, D))
        out = dict(dx=np.zeros((L, D)), dwq=np.zeros((D, D)), dwk=np.zeros((D, D)), dwv=np.zeros((D, D)),
                   dwo=np.zeros((D, D)), dw_score=np.zeros(D), dfeat=np.zeros_like(f))
        g = None if grad_out is None else np.ascontiguousarray(grad_out, np.float64)
        self._rc(self.lib.ref_linmix(C.c_int32(int(use_float)), C.c_uint64(L), C.c_uint64(D), _d(x), _d(wq),
                                     _d(wk), _d(wv), _d(wo), _d(ws), _d(f), C.byref(cfg),
                                     C.c_uint64(int(chunk_len)), None if g is None else _d(g), _d(y),
                                     *(_d(out[n]) for n in ("dx", "dwq", "dwk", "dwv", "dwo", "dw_score",
                                                            "dfeat"))))
        return y, (out if g is not None else None)

    def linear_mix_decode(self, x, wq, wk, wv, wo, w_score, feat, cfg, prompt, use_float=False):
        """SparseKvCache with LinearMixParams: forward_chunk(prompt), then generate_step per row."""
        x, wq, wk, wv, wo = (np.ascontiguousarray(a, np.float64) for a in (x, wq, wk, wv, wo))
        L, D = x.shape
        ws = np.ascontiguousarray(w_score if w_score is not None else np.zeros(D), np.float64)
        f = np.ascontiguousarray(feat, np.float64)
        y = np.zeros((L, D))
        self._rc(self.lib.ref_linmix_decode(C.c_int32(int(use_float)), C.c_uint64(L), C.c_uint64(D),
                                            C.c_uint64(prompt), _d(x), _d(wq), _d(wk), _d(wv), _d(wo), _d(ws),
                                            _d(f), C.byref(cfg), _d(y)))
        return y

    def bench_decode(self, units, threads, prompt, steps, p, k, window, seed=1):
        """Seconds for `steps` generate_step calls on each of `units` single-head
        caches prefilled with `prompt` rows (ref_bench_decode)."""
        secs = C.c_double()
        self._rc(self.lib.ref_bench_decode(C.c_uint64(units), C.c_uint64(threads), C.c_uint64(prompt),
                                           C.c_uint64(steps), C.c_uint64(p), C.c_double(k),
                                           C.c_uint64(window), C.c_uint64(seed), C.byref(secs)))
        return secs.value

def core_problem_via_reference(ref: Reference, Q, K, V, u_or_w, dO, *, kbudget, window,
                               key_mode="hard", mask_mode="soft", norm_mode="none",
                               slope_enabled=False, slope_eps=0.01,
                               slope_order="norm_then_slope", use_float=False):
    """Run the reference at core level with the identity-input trick.

    With x = I (L == D = H*p), Wq/Wk/Wv = Q/K/V, Wo = I and w_score = u_or_w the
    reference's projections return Q, K, V exactly, its raw scores are u_or_w,
    its dWq/dWk/dWv are dQ/dK/dV and its dw_score is the raw-score gradient.
    """
    L, H, p = Q.shape
    D = H * p
    assert L == D, "identity trick needs L == H*p"
    x = np.eye(L)
    cfg = ref_cfg(kbudget, window, heads=H, key_mode=key_mode, mask_mode=mask_mode,
                  slope_eps=slope_eps, slope_enabled=slope_enabled, norm_mode=norm_mode,
                  slope_order=slope_order)
    tape, grads = ref.attention(x, Q.reshape(L, D), K.reshape(L, D), V.reshape(L, D), np.eye(D),
                                u_or_w, cfg, use_float=use_float,
                                grad_out=None if dO is None else dO.reshape(L, D))
    return tape, grads
