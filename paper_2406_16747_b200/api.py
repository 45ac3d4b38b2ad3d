"""The reference's Python surface (``_sparsek``, proj/bindings/module.cpp:79-180),
re-implemented over the B200 kernels.

Same names, keyword arguments, return shapes and exception types as the
reference module, so ``import paper_2406_16747_b200 as sparsek`` is a drop-in for
``import sparsek``. Inputs are numpy arrays / sequences (copied to the GPU);
every computation runs in libsparsek_b200.so or cuBLAS (the D x D projections).
"""
from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _lib, ops
from ._lib import ArgumentError, ConfigError, NumericError, ShapeError

__version__ = "0.1.0"


def _dev():
    if not torch.cuda.is_available():
        raise _lib.CudaError("paper_2406_16747_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _vec(z, name):
    a = np.asarray(z, dtype=np.float64)
    if a.ndim != 1:
        raise ShapeError(f"{name}: expected a 1-D sequence")
    return a


def _tau_out(t):
    return float(t) if math.isfinite(t) else None


def _check_budget(k):
    if not (k > 0.0) or not math.isfinite(k):
        raise ArgumentError("KBudget: k must be positive and finite")


class PartialSortStats:
    """PartialSortStats (proj/include/sparsek/sparsek_op.hpp:42-45)."""

    def __init__(self):
        self.calls = 0
        self.fallbacks = 0

    def __repr__(self):
        return f"PartialSortStats(calls={self.calls}, fallbacks={self.fallbacks})"


def _solve_row(zz, k):
    zt = torch.from_numpy(zz).to(_dev()).view(1, -1)
    p, tau, uc, wc, fl = ops.sparsek_rows(zt, k)
    fl = int(fl[0])
    return {"p": p[0].cpu().numpy(), "tau": _tau_out(float(tau[0])), "u_count": int(uc[0]),
            "w_count": int(wc[0]), "degenerate": bool(fl & 1), "infeasible": bool(fl & 2)}


def _public(sol):
    return {key: sol[key] for key in ("p", "tau", "u_count", "w_count", "degenerate")}


def sparsek_partial(z, k, sort_cap, stats: PartialSortStats | None = None):
    """sparsek_partial (proj/src/sparsek_op.cpp:116-139): the solve restricted to
    the sort_cap largest values, falling back to the full solve when the cut
    cannot be certified. The device solver always evaluates the exact
    projection, which is what both branches of the reference return; ``stats``
    counts the calls and the reference's fallbacks — its truncated scan fails
    exactly when the accepted support reaches the cap (w_count >= sort_cap)."""
    k = float(k)
    zz = _vec(z, "sparsek_partial")
    if zz.size == 0:
        raise ArgumentError("sparsek_partial: empty input")
    _check_budget(k)
    if sort_cap < math.ceil(k):
        raise ArgumentError("sparsek_partial: sort_cap below ceil(k)")
    if stats is not None:
        stats.calls += 1
    if not np.all(np.isfinite(zz)):
        raise NumericError("sparsek_partial: non-finite input")
    sol = _solve_row(zz, k)
    if (stats is not None and not sol["infeasible"] and sort_cap < zz.size
            and sol["w_count"] >= sort_cap):
        stats.fallbacks += 1
    return _public(sol)


def sparsek(z, k, sort_cap=0):
    """Clamped-shift projection of z onto {0 <= p <= 1, sum p = k}
    (proj/src/sparsek_op.cpp:102-139). Returns {p, tau, u_count, w_count, degenerate}."""
    if sort_cap:
        return sparsek_partial(z, k, sort_cap)
    k = float(k)
    zz = _vec(z, "sparsek")
    if zz.size == 0:
        raise ArgumentError("sparsek: empty input")
    _check_budget(k)
    if not np.all(np.isfinite(zz)):
        raise NumericError("sparsek: non-finite input")
    return _public(_solve_row(zz, k))


def sparsek_st(z, k):
    """Straight-through pairing (proj/src/sparsek_op.cpp:167-172): the hard
    top-floor(k) forward and the soft solution as the gradient carrier.
    Returns {forward, backward_carrier}."""
    k = float(k)
    zz = _vec(z, "sparsek_st")
    if zz.size == 0:
        raise ArgumentError("sparsek: empty input")
    _check_budget(k)
    if not np.all(np.isfinite(zz)):
        raise NumericError("sparsek: non-finite input")
    carrier = _public(_solve_row(zz, k))
    return {"forward": topk_hard(zz, int(math.floor(k))), "backward_carrier": carrier}


def sparsek_jvp(z, k, v):
    """J(z) v = s * (v - mean_support(v)) (proj/src/sparsek_op.cpp:141-150)."""
    k = float(k)
    zz, vv = _vec(z, "sparsek_jvp"), _vec(v, "sparsek_jvp")
    if vv.size != zz.size:
        raise ShapeError("sparsek_jvp: v must match z")
    if zz.size == 0:
        raise ArgumentError("sparsek: empty input")
    _check_budget(k)
    if not np.all(np.isfinite(zz)):
        raise NumericError("sparsek: non-finite input")
    d = _dev()
    out = ops.sparsek_jvp_rows(torch.from_numpy(zz).to(d).view(1, -1), k,
                               torch.from_numpy(vv).to(d).view(1, -1))
    return out[0].cpu().numpy()


def topk_hard(z, k):
    """0/1 indicator of the k largest entries, ties to the lower index
    (proj/src/sparsek_op.cpp:152-165)."""
    zz = _vec(z, "topk_hard")
    out = ops.topk_hard_rows(torch.from_numpy(zz).to(_dev()).view(1, -1), int(k))
    return out[0].cpu().numpy()


from .stream import SelectionMask, Stream, stream_mask  # noqa: E402,F401  (device-resident StreamState)


def _mat(a, name):
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"{name}: expected a 2-D array")
    return m


def _attention_inputs(x, wq, wk, wv, wo, heads):
    x = _mat(x, "x")
    ws = [_mat(w, n) for w, n in ((wq, "wq"), (wk, "wk"), (wv, "wv"), (wo, "wo"))]
    L, D = x.shape
    for w in ws:
        if w.shape != (D, D):
            raise ShapeError("forward_chunk: projection shapes must be d_model x d_model")
    if heads <= 0:
        raise ConfigError("attention: heads must be positive")
    if D == 0 or D % heads:
        raise ConfigError("attention: d_model must be a positive multiple of heads")
    return x, ws


def _core_cfg(k, window, key_mode, mask_mode):
    if not math.isfinite(k) or k < 0.0:
        raise ConfigError("attention: k must be finite and >= 0")
    if window < 0:
        raise ConfigError("attention: window must be >= 0")
    if window == 0 and math.floor(k) < 1.0:
        raise ConfigError("attention: window + floor(k) must be >= 1 (only the linear mix can "
                          "run with neither)")
    if key_mode not in ("soft", "hard"):
        raise ArgumentError("key_mode must be 'soft' or 'hard'")
    if mask_mode not in ("soft", "straight_through"):
        raise ArgumentError("mask_mode must be 'soft' or 'straight_through'")
    return ops.AttnConfig(k=float(k), window=int(window), key_mode=key_mode, mask_mode=mask_mode)


_SIDE = {}
_FUSED_FRONT = os.environ.get("SKB_FUSED_FRONT", "0") == "1"


def _side_stream(device):
    """One side stream per device for K1 (kept, so no per-call creation)."""
    key = torch.device(device).index
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


def attention_torch(x, wq, wk, wv, wo, w_score, cfg: ops.AttnConfig, heads: int,
                    scoring: ops.ScoringConfig):
    """Differentiable x-level SparseK attention on device tensors:
    sparsek_attention (proj/include/sparsek/attention.hpp:81-85) as torch ops.
    x: [B, L, D]; W*: [D, D]; w_score: [D]. Projections are cuBLAS GEMMs; the
    score, selection, attention and their backward are libsparsek_b200 kernels."""
    B, L, D = x.shape
    p = D // heads
    if _FUSED_FRONT and ops.proj_supported(x, wq) and (cfg.k == 0.0 or w_score is not None):
        # opt-in (SKB_FUSED_FRONT=1; bf16, d_model % 256 == 0): the hand-written
        # CTA-pair tcgen05 projection GEMM with the score formed from the same x
        # rows and its Welford streaming under it. At cfg3 it measures 3.48 ms
        # against 3.12 ms for cuBLAS + K1 on a side stream,
        # so the library front stays the default.
        q, k, v, u = ops.ProjScoreFn.apply(x, wq, wk, wv, w_score if cfg.k > 0.0 else None, scoring)
        if u is None:
            u = torch.zeros((B, L), dtype=torch.float64, device=x.device)
        hc = ops.sparsek_attention_core(q.view(B, L, heads, p), k.view(B, L, heads, p), v.view(B, L, heads, p),
                                        u, cfg)
        return hc.reshape(B, L, D) @ wo, hc
    main = torch.cuda.current_stream(x.device)
    side = _side_stream(x.device) if cfg.k > 0.0 else None
    if side is not None:  # K1's serial Welford chain runs under the projection GEMMs
        side.wait_stream(main)
    q = (x @ wq).view(B, L, heads, p)
    k = (x @ wk).view(B, L, heads, p)
    v = (x @ wv).view(B, L, heads, p)
    if cfg.k > 0.0:
        with torch.cuda.stream(side):
            u = ops.score_tokens(x, w_score, scoring)
        main.wait_stream(side)
        x.record_stream(side)
        u.record_stream(main)
    else:
        u = torch.zeros((B, L), dtype=torch.float64, device=x.device)
    hc = ops.sparsek_attention_core(q, k, v, u, cfg)
    return hc.reshape(B, L, D) @ wo, hc


def attention(x, wq, wk, wv, wo, w_score, k, window, heads=1, key_mode="hard", mask_mode="soft",
              slope_eps=0.01, slope_enabled=True):
    """Causal attention where each query sees its sliding window plus the top-k
    scored positions that already left it (the reference's ``attention``)."""
    x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
    cfg = _core_cfg(float(k), int(window), key_mode, mask_mode)
    L, D = x.shape
    wsc = _vec(w_score, "w_score")
    if cfg.k > 0.0 and wsc.size != D:
        raise ConfigError("attention: w_score length must equal d_model")
    if not (slope_eps > 0.0):
        raise ArgumentError("ScoringParams: slope_eps must be positive")
    if not np.all(np.isfinite(wsc)):
        raise NumericError("ScoringParams: non-finite w_score")
    d = _dev()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled))
    with torch.no_grad():
        y, _ = attention_torch(t(x).view(1, L, D), t(wq), t(wk), t(wv), t(wo),
                               t(wsc) if cfg.k > 0.0 else None, cfg, heads, sc)
    return y[0].cpu().numpy()


def attention_grads(x, wq, wk, wv, wo, w_score, k, window, grad_out, heads=1, key_mode="hard",
                    mask_mode="soft", slope_eps=0.01, slope_enabled=True,
                    norm_mode="timestep_norm", slope_order="norm_then_slope", chunk_len=0):
    """Forward + sparsek_attention_backward (proj/src/attention.cpp:214-575):
    returns (y, {dx, dwq, dwk, dwv, dwo, dw_score}) as float64 numpy arrays.
    chunk_len > 0 is chunked_forward's training (Algorithm 3,
    proj/src/cache.cpp:548-563): the same outputs, and gradients that never
    cross to the left of a chunk start (proj/src/attention.cpp:228-234)."""
    x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
    if int(chunk_len) < 0:
        raise ArgumentError("chunked_forward: chunk_len must be positive")
    cfg = _core_cfg(float(k), int(window), key_mode, mask_mode)
    if chunk_len:
        cfg = ops.AttnConfig(k=cfg.k, window=cfg.window, key_mode=cfg.key_mode,
                             mask_mode=cfg.mask_mode, chunk_len=int(chunk_len))
    L, D = x.shape
    wsc = _vec(w_score, "w_score")
    d = _dev()
    leaf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d).requires_grad_(True)
    xt, wqt, wkt, wvt, wot, wst = (leaf(a) for a in (x, wq, wk, wv, wo, wsc))
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled),
                           norm_mode=norm_mode, slope_order=slope_order, chunk_len=int(chunk_len))
    y, _ = attention_torch(xt.view(1, L, D), wqt, wkt, wvt, wot, wst, cfg, heads, sc)
    y.backward(torch.from_numpy(np.ascontiguousarray(grad_out, np.float64)).to(d).view(1, L, D))
    g = lambda t: (t.grad.cpu().numpy() if t.grad is not None else np.zeros(tuple(t.shape)))
    return y[0].detach().cpu().numpy(), dict(dx=g(xt), dwq=g(wqt), dwk=g(wkt), dwv=g(wvt),
                                             dwo=g(wot), dw_score=g(wst))


def _lm_inputs(x, wq, wk, wv, wo, w_score, feat, k, window, heads, slope_eps):
    x, ws = _attention_inputs(x, wq, wk, wv, wo, heads)
    if not math.isfinite(k) or k < 0.0:
        raise ConfigError("attention: k must be finite and >= 0")
    if window < 0:
        raise ConfigError("attention: window must be >= 0")
    L, D = x.shape
    p = D // heads
    wsc = _vec(w_score, "w_score") if w_score is not None else np.zeros(0)
    if k > 0.0 and wsc.size != D:
        raise ConfigError("attention: w_score length must equal d_model")
    if not (slope_eps > 0.0):
        raise ArgumentError("ScoringParams: slope_eps must be positive")
    f = np.asarray(feat, dtype=np.float64)
    if f.ndim != 3 or f.shape[0] != heads:
        raise ShapeError("forward_chunk: one feature map per head")
    if f.shape[1:] != (p, p):
        raise ShapeError("forward_chunk: feature maps are head_dim x head_dim")
    cfg = ops.AttnConfig(k=float(k), window=int(window), linear_mix=True)
    return x, ws, wsc, f, cfg


def linear_mix_torch(x, wq, wk, wv, wo, w_score, feat, cfg: ops.AttnConfig, heads: int,
                     scoring: ops.ScoringConfig):
    """Differentiable x-level linear_mix_attention (proj/include/sparsek/
    attention.hpp:93-99) on device tensors: x [B, L, D], feat [H, p, p]."""
    B, L, D = x.shape
    p = D // heads
    if scoring.norm_mode != "timestep_norm":
        raise ConfigError("linear mix requires timestep normalization; raw scores make the linear "
                          "branch blow up")
    q = (x @ wq).view(B, L, heads, p)
    k = (x @ wk).view(B, L, heads, p)
    v = (x @ wv).view(B, L, heads, p)
    if cfg.k > 0.0:
        u = ops.score_tokens(x, w_score, scoring)
    else:
        u = torch.zeros((B, L), dtype=torch.float64, device=x.device)
    hc = ops.linear_mix_core(q, k, v, u, feat, cfg)
    return hc.reshape(B, L, D) @ wo, hc


def linear_mix_attention(x, wq, wk, wv, wo, w_score, feat, k, window, heads=1, slope_eps=0.01,
                         slope_enabled=True):
    """linear_mix_attention (proj/include/sparsek/attention.hpp:93-99; Appendix
    B.1): the SparseK snapshot's exact attention mixed with positive-feature
    linear attention over every causal position; feat: [H, p, p] (one feature
    map per head). float64 in and out, like the reference's double path."""
    x, (wq, wk, wv, wo), wsc, f, cfg = _lm_inputs(x, wq, wk, wv, wo, w_score, feat, k, window, heads,
                                                   slope_eps)
    L, D = x.shape
    d = _dev()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled))
    with torch.no_grad():
        y, _ = linear_mix_torch(t(x).view(1, L, D), t(wq), t(wk), t(wv), t(wo),
                                t(wsc) if cfg.k > 0.0 else None, t(f), cfg, heads, sc)
    return y[0].cpu().numpy()


def linear_mix_attention_grads(x, wq, wk, wv, wo, w_score, feat, k, window, grad_out, heads=1,
                               slope_eps=0.01, slope_enabled=True, chunk_len=0):
    """linear_mix_attention + sparsek_attention_backward with LinearMixParams
    (proj/src/attention.cpp:317-445, 519-549): (y, {dx, dwq, dwk, dwv, dwo,
    dw_score, dfeat}) as float64 numpy arrays."""
    x, (wq, wk, wv, wo), wsc, f, cfg = _lm_inputs(x, wq, wk, wv, wo, w_score, feat, k, window, heads,
                                                   slope_eps)
    if chunk_len:
        cfg = ops.AttnConfig(k=cfg.k, window=cfg.window, linear_mix=True, chunk_len=int(chunk_len))
    L, D = x.shape
    d = _dev()
    leaf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d).requires_grad_(True)
    xt, wqt, wkt, wvt, wot, ft = (leaf(a) for a in (x, wq, wk, wv, wo, f))
    wst = leaf(wsc) if cfg.k > 0.0 else None
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled),
                           chunk_len=int(chunk_len))
    y, _ = linear_mix_torch(xt.view(1, L, D), wqt, wkt, wvt, wot, wst, ft, cfg, heads, sc)
    y.backward(torch.from_numpy(np.ascontiguousarray(grad_out, np.float64)).to(d).view(1, L, D))
    g = lambda t: (t.grad.cpu().numpy() if t is not None and t.grad is not None
                   else np.zeros(tuple(t.shape) if t is not None else (D,)))
    return y[0].detach().cpu().numpy(), dict(dx=g(xt), dwq=g(wqt), dwk=g(wkt), dwv=g(wvt), dwo=g(wot),
                                             dw_score=g(wst) if wst is not None else np.zeros(D),
                                             dfeat=g(ft))


def chunked_forward(x, chunk_len, wq, wk, wv, wo, w_score, k, window, heads=1, key_mode="hard",
                    mask_mode="soft", slope_eps=0.01, slope_enabled=True):
    """chunked_forward (proj/src/cache.cpp:548-563, Algorithm 3): the sequence is
    fed chunk by chunk into ONE recurrent cache whose state between chunks is
    the constant-(floor(k)+w) retained K/V rows, the stream survivors and the
    carried TimestepNormState — DecodeSession.forward_chunk. The first chunk
    runs the batch kernels, each later chunk continues the state row by row
    (generate_step's order). The output equals the unchunked forward
    (proj/tests/test_cache.cpp:34-64)."""
    if int(chunk_len) <= 0:
        raise ArgumentError("chunked_forward: chunk_len must be positive")
    x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
    cfg = _core_cfg(float(k), int(window), key_mode, mask_mode)
    L, D = x.shape
    wsc = _vec(w_score, "w_score")
    if cfg.k > 0.0 and wsc.size != D:
        raise ConfigError("attention: w_score length must equal d_model")
    if not (slope_eps > 0.0):
        raise ArgumentError("ScoringParams: slope_eps must be positive")
    d = _dev()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled))
    sess = DecodeSession(t(wq), t(wk), t(wv), t(wo), t(wsc) if cfg.k > 0.0 else None, cfg, heads, 1,
                         max_len=L, scoring=sc, dtype=torch.float64)
    xt = t(x).view(1, L, D)
    outs = [sess.forward_chunk(xt[:, c0:c0 + int(chunk_len)]) for c0 in range(0, L, int(chunk_len))]
    return torch.cat(outs, 1)[0].cpu().numpy()


class DecodeSession:
    """x-level generation over a batch of B sequences: SparseKvCache::forward_chunk
    on a prompt followed by generate_step per new row (proj/src/cache.cpp:195-230,
    570-577). Device tensors throughout: projections are cuBLAS GEMMs, the score
    continues a per-sequence TimestepNormState on the device (skb_score_continue),
    the prompt's outputs come from the batch kernels (K2/K3; the same outputs
    forward_chunk gives, proj/tests/test_cache.cpp:34-64) and every step is one
    skb_cache_step (K5) over the constant-(floor(k)+w) pool.

    x rows are [B, D] (step) or [B, n, D] (prefill) in the session dtype; w* are
    [D, D], w_score [D]."""

    def __init__(self, wq, wk, wv, wo, w_score, cfg: ops.AttnConfig, heads: int, batch: int,
                 max_len: int, scoring: ops.ScoringConfig = ops.ScoringConfig(), dtype=None, feat=None):
        """feat [H, p, p] (LinearMixParams): the linear-attention mix (Appendix B.1),
        float32/float64 sessions; its prefix state is carried by the cache."""
        self.wq, self.wk, self.wv, self.wo = wq, wk, wv, wo
        self.feat = feat
        if feat is not None:
            import dataclasses

            cfg = cfg if cfg.linear_mix else dataclasses.replace(cfg, linear_mix=True)
            if scoring.norm_mode != "timestep_norm":
                raise ConfigError("linear mix requires timestep normalization; raw scores make the linear "
                                  "branch blow up")
        D = wq.shape[0]
        if D % heads:
            raise ConfigError("attention: d_model must be a positive multiple of heads")
        self.D, self.H, self.p, self.B = D, int(heads), D // int(heads), int(batch)
        self.cfg, self.sc = cfg, scoring
        self.dtype = dtype or wq.dtype
        self.w_score = w_score
        if cfg.k > 0.0 and (w_score is None or w_score.shape != (D,)):
            raise ConfigError("attention: w_score length must equal d_model")
        self.state = torch.zeros((self.B, 3), dtype=torch.float64, device=wq.device)
        self.cache = ops.DecodeCache(self.B, self.H, self.p, cfg, max_len, dtype=self.dtype,
                                     device=wq.device)
        self.t = 0

    def _proj_score(self, x):
        B, n, D = x.shape
        q, k, v = ((x @ w).view(B, n, self.H, self.p) for w in (self.wq, self.wk, self.wv))
        if self.cfg.k > 0.0:
            _, u = ops.score_continue(x, self.w_score, self.sc, self.state)
        else:
            u = torch.zeros((B, n), dtype=torch.float64, device=x.device)
        return q, k, v, u

    @torch.no_grad()
    def forward_chunk(self, x):
        """SparseKvCache::forward_chunk (proj/src/cache.cpp:181-400) on rows
        x [B, n, D] that continue every sequence; returns y [B, n, D]. A fresh
        cache runs the batch kernels over the chunk (prefill); a non-empty one
        continues its carried state one generate_step per row (the reference's
        row order), with the chunk's projections and scores done in one pass."""
        B, n, D = x.shape
        if n < 1:
            raise ShapeError("forward_chunk: empty chunk")
        if self.t == 0 and n > 1:
            return self.prefill(x)
        q, k, v, u = self._proj_score(x)
        outs = []
        for r in range(n):
            qr, kr, vr, ur = (t[:, r].contiguous() for t in (q, k, v, u))
            if self.feat is not None:
                outs.append(self.cache.linmix_step(qr, kr, vr, ur, ops.linmix_phi(qr, self.feat),
                                                   ops.linmix_phi(kr, self.feat)))
            else:
                outs.append(self.cache.step(qr, kr, vr, ur))
            self.t += 1
        return torch.stack(outs, 1).reshape(B, n, D) @ self.wo

    @torch.no_grad()
    def prefill(self, x):
        """forward_chunk on a prompt x [B, n, D] of a fresh cache (the batch
        kernels); on a non-empty cache this is forward_chunk's continuation.
        Returns y [B, n, D]."""
        if self.t:
            return self.forward_chunk(x)
        B, n, D = x.shape
        q, k, v, u = self._proj_score(x)
        q, k, v, u = q.contiguous(), k.contiguous(), v.contiguous(), u.contiguous()
        if self.feat is not None:  # the mixture readout over the prompt (batch kernels)
            hc, _, _ = ops.linmix_fwd(q, k, v, u, self.feat, self.cfg)
        else:
            hc = ops.sparsek_attention_core(q, k, v, u, self.cfg)
        self.cache.prefill(k, v, u)
        if self.feat is not None:
            self.cache.linmix_prefill(v, ops.linmix_phi(k, self.feat))
        self.t = n
        return hc.reshape(B, n, D) @ self.wo

    def snapshot(self, b=0):
        """The reference's cache snapshot payload of sequence b (cache, stream,
        TimestepNormState): SparseKvCache::serialize, proj/src/cache.cpp:416-475."""
        st = self.state[b].tolist()
        return self.cache.snapshot(b, norm_state=st)

    def restore(self, blob, b=0):
        """Resume sequence b from a snapshot payload (ours or the reference's)."""
        ns = self.cache.restore(blob, b)
        self.state[b] = torch.tensor(ns, dtype=torch.float64, device=self.state.device)
        self.t = max(self.t, int(self.cache.state(b)["seen"]))

    @torch.no_grad()
    def step(self, x_row):
        """generate_step: x_row [B, D] -> y [B, D]."""
        return self.forward_chunk(x_row.view(self.B, 1, self.D)).reshape(self.B, self.D)


def save_cache_snapshot(path, payload):
    """save_cache_snapshot's file format (proj/src/cache.cpp:579-595): "SPKC",
    u16 version 1, u64 payload length (little endian), payload."""
    import struct

    with open(path, "wb") as f:
        f.write(b"SPKC" + struct.pack("<HQ", 1, len(payload)) + payload)


def load_cache_snapshot(path):
    """The payload of a save_cache_snapshot file (proj/src/cache.cpp:597-618)."""
    import struct

    from ._lib import IoError

    with open(path, "rb") as f:
        head = f.read(14)
        if len(head) < 4 or head[:4] != b"SPKC":
            raise IoError(f"not a cache snapshot: {path}")
        if len(head) < 14:
            raise IoError("cache snapshot: truncated header")
        ver, n = struct.unpack("<HQ", head[4:])
        if ver != 1:
            raise IoError("cache snapshot: unsupported version")
        payload = f.read(n)
        if len(payload) != n:
            raise IoError("cache snapshot: truncated payload")
        return payload


def dense_attention(x, wq, wk, wv, wo, heads=1):
    """Quadratic causal softmax attention (proj/src/attention.cpp:76-111): the
    SparseK kernels with a budget covering every position (all gates 1)."""
    x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
    L, D = x.shape
    p = D // heads
    d = _dev()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
    xt = t(x)
    cfg = ops.AttnConfig(k=float(L + 1), window=1)
    q, kk, v = ((xt @ t(w)).view(1, L, heads, p) for w in (wq, wk, wv))
    u = torch.zeros((1, L), dtype=torch.float64, device=d)
    o, _, _ = ops.attn_fwd(q.contiguous(), kk.contiguous(), v.contiguous(), u, cfg)
    return (o.reshape(L, D) @ t(wo)).cpu().numpy()


def dense_attention_grads(x, wq, wk, wv, wo, grad_out, heads=1):
    """dense_causal_attention + dense_causal_attention_backward
    (proj/src/attention.cpp:76-205): returns (y, {dx, dwq, dwk, dwv, dwo}) as
    float64 numpy arrays. The attention core is the SparseK kernels with a
    budget covering every position (tau = -inf, every gate 1) and constant
    scores, so no gradient reaches a score."""
    x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
    L, D = x.shape
    p = D // heads
    d = _dev()
    leaf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d).requires_grad_(True)
    xt, wqt, wkt, wvt, wot = (leaf(a) for a in (x, wq, wk, wv, wo))
    cfg = ops.AttnConfig(k=float(L + 1), window=1)
    q, kk, v = ((xt @ w).view(1, L, heads, p) for w in (wqt, wkt, wvt))
    u = torch.zeros((1, L), dtype=torch.float64, device=d)
    hc = ops.sparsek_attention_core(q, kk, v, u, cfg)
    y = hc.reshape(L, D) @ wot
    y.backward(torch.from_numpy(np.ascontiguousarray(grad_out, np.float64)).to(d))
    return y.detach().cpu().numpy(), dict(dx=xt.grad.cpu().numpy(), dwq=wqt.grad.cpu().numpy(),
                                          dwk=wkt.grad.cpu().numpy(), dwv=wvt.grad.cpu().numpy(),
                                          dwo=wot.grad.cpu().numpy())


def attention_with_tape(x, wq, wk, wv, wo, w_score, k, window, heads=1, key_mode="hard",
                        mask_mode="soft", slope_eps=0.01, slope_enabled=True,
                        norm_mode="timestep_norm", slope_order="norm_then_slope", chunk_len=0):
    """sparsek_attention with an AttnTape (proj/include/sparsek/attention.hpp:81-85):
    returns (y, tape); the tape stays on the device and feeds
    ``attention_backward``. Inputs are numpy (float64, like the bindings) or
    device tensors (their dtype is kept)."""
    from . import tape as tp

    if isinstance(x, torch.Tensor):
        d = x.device
        conv = lambda a: a
    else:
        x, (wq, wk, wv, wo) = _attention_inputs(x, wq, wk, wv, wo, heads)
        d = _dev()
        conv = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(d)
    cfg = _core_cfg(float(k), int(window), key_mode, mask_mode)
    if chunk_len:
        cfg = ops.AttnConfig(k=cfg.k, window=cfg.window, key_mode=cfg.key_mode, mask_mode=cfg.mask_mode,
                             chunk_len=int(chunk_len))
    params = tp.AttnParams(conv(wq), conv(wk), conv(wv), conv(wo))
    sc = ops.ScoringConfig(slope_eps=float(slope_eps), slope_enabled=bool(slope_enabled),
                           norm_mode=norm_mode, slope_order=slope_order, chunk_len=int(chunk_len))
    ws = conv(w_score) if (w_score is not None and cfg.k > 0.0) else None
    tape = tp.AttnTape()
    y = tp.forward(conv(x), params, ws, sc, cfg, int(heads), tape)
    tape.params, tape.w_score, tape.scoring = params, ws, sc
    return (y if isinstance(x, torch.Tensor) else y.cpu().numpy()), tape


def attention_backward(tape, grad_out):
    """sparsek_attention_backward (proj/src/attention.cpp:214-575) from a tape
    made by ``attention_with_tape``: {dx, dwq, dwk, dwv, dwo, dw_score}."""
    from . import tape as tp

    host = not isinstance(grad_out, torch.Tensor)
    g = torch.from_numpy(np.ascontiguousarray(grad_out, np.float64)).to(tape.x.device) if host else grad_out
    out = tp.backward(tape, g, tape.params, tape.w_score, tape.scoring)
    if tape.x.shape[0] == 1:
        out["dx"] = out["dx"][0]
    return {k: v.cpu().numpy() for k, v in out.items()} if host else out
