"""Torch-level entry points over the C ABI (device tensors in, device tensors out).

Layout: q/k/v/o/dO are [B, L, H, p] (the reference's per-sequence [L, D] with
head h in columns [h*p, (h+1)*p), proj/include/sparsek/attention.hpp:36);
scores u are float64 [B, L] (proj/include/sparsek/selection.hpp:72-74).
All work runs in libsparsek_b200.so on the current CUDA stream.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import AttnDesc, Scoring, SelectLayout, check

_DT = {torch.float32: _lib.SKB_F32, torch.bfloat16: _lib.SKB_BF16, torch.float64: _lib.SKB_F64}


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _on_device(fn):
    """Run `fn` with its first CUDA tensor argument's device current, so the
    launches and torch's current stream both belong to that device."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kw):
        for a in list(args) + list(kw.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                with torch.cuda.device(a.device):
                    return fn(*args, **kw)
        return fn(*args, **kw)

    return wrapped


@dataclass(frozen=True)
class AttnConfig:
    """AttnConfig (proj/include/sparsek/attention.hpp:18-32) at the core level."""
    k: float = 8.0
    window: int = 8
    scale: float = 0.0
    key_mode: str = "hard"       # "hard" | "soft"
    mask_mode: str = "soft"      # "soft" | "straight_through"
    force_gather: bool = False   # BF16 on the CUDA-core gather kernels
    chunk_len: int = 0           # chunked_forward (Algorithm 3): backward stop-grad at chunk starts
    linear_mix: bool = False     # Appendix B.1 (linear_mix_attention): window = floor(k) = 0 allowed

    def key_code(self):
        if self.key_mode not in ("hard", "soft"):
            raise _lib.ArgumentError("key_mode must be 'soft' or 'hard'")
        return int(self.key_mode == "soft")

    def mask_code(self):
        if self.mask_mode not in ("soft", "straight_through"):
            raise _lib.ArgumentError("mask_mode must be 'soft' or 'straight_through'")
        return int(self.mask_mode == "straight_through")


def make_desc(B, L, H, p, cfg: AttnConfig, dtype: torch.dtype) -> AttnDesc:
    if dtype not in _DT:
        raise _lib.ArgumentError(f"unsupported dtype {dtype}")
    flags = (_lib.SKB_FLAG_FORCE_GATHER if cfg.force_gather else 0) | \
        (_lib.SKB_FLAG_LINEAR_MIX if cfg.linear_mix else 0)
    if cfg.chunk_len < 0:
        raise _lib.ArgumentError("chunked_forward: chunk_len must be positive")
    return AttnDesc(int(B), int(L), int(H), int(p), float(cfg.k), int(cfg.window),
                    float(cfg.scale), cfg.key_code(), cfg.mask_code(), _DT[dtype], flags,
                    int(cfg.chunk_len))


def _check_qkv(q, k, v):
    if q.dim() != 4:
        raise _lib.ShapeError("q/k/v must be [B, L, H, p]")
    if k.shape != q.shape or v.shape != q.shape:
        raise _lib.ShapeError("q, k, v must share one [B, L, H, p] shape")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise _lib.ArgumentError("q/k/v must be CUDA tensors")
    if not (q.dtype == k.dtype == v.dtype):
        raise _lib.ArgumentError("q/k/v dtypes differ")
    for t in (q, k, v):
        if not t.is_contiguous():
            raise _lib.ArgumentError("q/k/v must be contiguous")


class Selection:
    """Device-resident output of K2 (skb_select) for one batch of sequences."""

    def __init__(self, desc: AttnDesc, ws: torch.Tensor, layout: SelectLayout):
        self.desc, self.ws, self.layout = desc, ws, layout

    def _view(self, off, dtype, count):
        esz = torch.tensor([], dtype=dtype).element_size()
        return self.ws[off: off + count * esz].view(dtype)

    @property
    def leave(self):
        B, L = self.desc.batch, self.desc.seq_len
        return self._view(self.layout.leave, torch.int32, B * L).view(B, L)

    @property
    def tau(self):
        """Threshold after each push time t (float64 [B, L]; entries t >= L-w unused)."""
        B, L = self.desc.batch, self.desc.seq_len
        return self._view(self.layout.tau, torch.float64, B * L).view(B, L)

    @property
    def nfrac(self):
        B, L = self.desc.batch, self.desc.seq_len
        return self._view(self.layout.nfrac, torch.int32, B * L).view(B, L)

    @property
    def qb_count(self):
        B, n = self.desc.batch, self.layout.nqb
        return self._view(self.layout.qb_count, torch.int32, B * n).view(B, n)

    @property
    def qb_list(self):
        B, n, c = self.desc.batch, self.layout.nqb, self.layout.qb_cap
        return self._view(self.layout.qb_list, torch.int32, B * n * c).view(B, n, c)

    def tau_per_query(self):
        """tau each query froze (float64 [B, L], -inf before the first push)."""
        B, L, w = self.desc.batch, self.desc.seq_len, self.desc.window
        out = torch.full((B, L), -math.inf, dtype=torch.float64, device=self.ws.device)
        if L > w:
            out[:, w:] = self.tau[:, : L - w]
        return out


def _scores(u, B, L, device):
    """u as a contiguous float64 [B, L] tensor on `device` (the kernels read it raw)."""
    if u.shape != (B, L):
        raise _lib.ShapeError("u must be [B, L]")
    if u.dtype != torch.float64 or u.device != device:
        raise _lib.ArgumentError("u must be a float64 tensor on the q/k/v device")
    return u.contiguous()


def select(u: torch.Tensor, cfg: AttnConfig, heads=1, head_dim=1, dtype=torch.float32,
           desc: AttnDesc | None = None) -> Selection:
    """K2: prefix tau and top-floor(k) retention intervals for u [B, L] float64."""
    if u.dim() != 2 or u.dtype != torch.float64 or not u.is_cuda:
        raise _lib.ArgumentError("u must be a CUDA float64 [B, L] tensor")
    u = u.contiguous()
    B, L = u.shape
    if desc is None:
        desc = make_desc(B, L, heads, head_dim, cfg, dtype)
    lay = SelectLayout()
    check(_lib.load().skb_select_layout_of(desc, lay))
    with torch.cuda.device(u.device):
        ws = torch.empty(lay.total_bytes, dtype=torch.uint8, device=u.device)
        check(_lib.load().skb_select(desc, u.data_ptr(), ws.data_ptr(), _stream()))
    return Selection(desc, ws, lay)


def attn_fwd(q, k, v, u, cfg: AttnConfig, sel: Selection | None = None):
    """K3. Returns (o [B,L,H,p], lse float64 [B,H,L], selection)."""
    _check_qkv(q, k, v)
    B, L, H, p = q.shape
    u = _scores(u, B, L, q.device)
    desc = make_desc(B, L, H, p, cfg, q.dtype)
    with torch.cuda.device(q.device):
        if sel is None:
            sel = select(u, cfg, desc=desc)
        o = torch.empty_like(q)
        lse = torch.empty((B, H, L), dtype=torch.float64, device=q.device)
        check(_lib.load().skb_attn_fwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), u.data_ptr(),
                                       sel.ws.data_ptr(), o.data_ptr(), lse.data_ptr(), _stream()))
    return o, lse, sel


def attn_bwd(q, k, v, o, do, lse, u, sel: Selection, cfg: AttnConfig, ws=None):
    """K4 + selection pullback. Returns (dq, dk, dv, du float64 [B, L])."""
    _check_qkv(q, k, v)
    B, L, H, p = q.shape
    u = _scores(u, B, L, q.device)
    if lse.shape != (B, H, L) or lse.dtype != torch.float64 or not lse.is_contiguous():
        raise _lib.ArgumentError("attn_bwd: lse must be a contiguous float64 [B, H, L] tensor")
    if o is not None and (o.shape != q.shape or o.dtype != q.dtype or not o.is_contiguous()):
        raise _lib.ArgumentError("attn_bwd: o must be contiguous with q's shape and dtype")
    desc = make_desc(B, L, H, p, cfg, q.dtype)
    do = do.contiguous()
    if do.dtype != q.dtype:
        do = do.to(q.dtype)
    lib = _lib.load()
    with torch.cuda.device(q.device):
        if ws is None:
            n = C_size()
            check(lib.skb_attn_bwd_workspace_size(desc, n))
            ws = torch.empty(n.value, dtype=torch.uint8, device=q.device)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        du = torch.empty((B, L), dtype=torch.float64, device=q.device)
        check(lib.skb_attn_bwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), _ptr(o), do.data_ptr(),
                               lse.data_ptr(), u.data_ptr(), sel.ws.data_ptr(), dq.data_ptr(),
                               dk.data_ptr(), dv.data_ptr(), du.data_ptr(), ws.data_ptr(), _stream()))
    return dq, dk, dv, du


def bwd_workspace(q, cfg: AttnConfig):
    B, L, H, p = q.shape
    desc = make_desc(B, L, H, p, cfg, q.dtype)
    n = C_size()
    check(_lib.load().skb_attn_bwd_workspace_size(desc, n))
    return torch.empty(n.value, dtype=torch.uint8, device=q.device)


def C_size():
    import ctypes

    return ctypes.c_size_t()


class SparseKAttentionFn(torch.autograd.Function):
    """Core SparseK attention with its closed-form backward (q, k, v, u) -> o."""

    @staticmethod
    def forward(ctx, q, k, v, u, cfg: AttnConfig):
        q, k, v, u = q.contiguous(), k.contiguous(), v.contiguous(), u.contiguous()
        o, lse, sel = attn_fwd(q, k, v, u, cfg)
        ctx.save_for_backward(q, k, v, o, lse, u)
        ctx.sel, ctx.cfg = sel, cfg
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse, u = ctx.saved_tensors
        dq, dk, dv, du = attn_bwd(q, k, v, o, do, lse, u, ctx.sel, ctx.cfg)
        return dq, dk, dv, du, None


def sparsek_attention_core(q, k, v, u, cfg: AttnConfig):
    return SparseKAttentionFn.apply(q, k, v, u, cfg)


# ---------------------------------------------------------------- linear-attention mix

def _linmix_ws(desc, device):
    n = C_size()
    check(_lib.load().skb_linmix_workspace_size(desc, n))
    return torch.empty(n.value, dtype=torch.uint8, device=device)


def _feat(feat, H, p, device):
    if feat.shape != (H, p, p):
        raise _lib.ShapeError("forward_chunk: feature maps are head_dim x head_dim (one per head)")
    return feat.to(device=device, dtype=torch.float64).contiguous()


def _lm_cfg(cfg: AttnConfig) -> AttnConfig:
    import dataclasses

    return cfg if cfg.linear_mix else dataclasses.replace(cfg, linear_mix=True)


def linmix_fwd(q, k, v, u, feat, cfg: AttnConfig, sel: Selection | None = None):
    """Linear-attention mix forward (skb_linmix_fwd): q/k/v [B, L, H, p] float32
    or float64, u [B, L] float64, feat [H, p, p]. Returns (o, den [B, H, L],
    selection)."""
    _check_qkv(q, k, v)
    cfg = _lm_cfg(cfg)
    B, L, H, p = q.shape
    u = _scores(u, B, L, q.device)
    desc = make_desc(B, L, H, p, cfg, q.dtype)
    f = _feat(feat, H, p, q.device)
    with torch.cuda.device(q.device):
        if sel is None:
            sel = select(u, cfg, desc=desc)
        o = torch.empty_like(q)
        den = torch.empty((B, H, L), dtype=torch.float64, device=q.device)
        ws = _linmix_ws(desc, q.device)
        check(_lib.load().skb_linmix_fwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), u.data_ptr(),
                                         sel.ws.data_ptr(), f.data_ptr(), o.data_ptr(), den.data_ptr(),
                                         ws.data_ptr(), _stream()))
    return o, den, sel


def linmix_bwd(q, k, v, u, feat, den, do, sel: Selection, cfg: AttnConfig):
    """Returns (dq, dk, dv, du [B, L] float64, dfeat [H, p, p] float64)."""
    _check_qkv(q, k, v)
    cfg = _lm_cfg(cfg)
    B, L, H, p = q.shape
    u = _scores(u, B, L, q.device)
    desc = make_desc(B, L, H, p, cfg, q.dtype)
    f = _feat(feat, H, p, q.device)
    if den.shape != (B, H, L) or den.dtype != torch.float64 or not den.is_contiguous():
        raise _lib.ArgumentError("linear mix backward: den must be a contiguous float64 [B, H, L] tensor")
    do = do.contiguous().to(q.dtype)
    with torch.cuda.device(q.device):
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        du = torch.empty((B, L), dtype=torch.float64, device=q.device)
        dfeat = torch.empty((H, p, p), dtype=torch.float64, device=q.device)
        ws = _linmix_ws(desc, q.device)
        check(_lib.load().skb_linmix_bwd(desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), u.data_ptr(),
                                         sel.ws.data_ptr(), f.data_ptr(), den.data_ptr(), do.data_ptr(),
                                         dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), du.data_ptr(),
                                         dfeat.data_ptr(), ws.data_ptr(), _stream()))
    return dq, dk, dv, du, dfeat


@_on_device
def linmix_phi(z, feat):
    """phi(z) = elu(F_h z) + 1 of rows z [..., H, p] (float32/float64) -> float64."""
    H, p = z.shape[-2], z.shape[-1]
    z = z.contiguous()
    f = _feat(feat, H, p, z.device)
    out = torch.empty(z.shape, dtype=torch.float64, device=z.device)
    rows = z.numel() // (H * p)
    check(_lib.load().skb_linmix_phi(rows, H, p, _DT[z.dtype], z.data_ptr(), f.data_ptr(), out.data_ptr(),
                                     _stream()))
    return out


class LinearMixFn(torch.autograd.Function):
    """(q, k, v, u, feat) -> o for the linear-attention mix, with its backward."""

    @staticmethod
    def forward(ctx, q, k, v, u, feat, cfg: AttnConfig):
        q, k, v, u = q.contiguous(), k.contiguous(), v.contiguous(), u.contiguous()
        o, den, sel = linmix_fwd(q, k, v, u, feat, cfg)
        ctx.save_for_backward(q, k, v, u, feat, den)
        ctx.sel, ctx.cfg = sel, cfg
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, u, feat, den = ctx.saved_tensors
        dq, dk, dv, du, dfeat = linmix_bwd(q, k, v, u, feat, den, do, ctx.sel, ctx.cfg)
        return dq, dk, dv, du, dfeat.to(feat.dtype), None


def linear_mix_core(q, k, v, u, feat, cfg: AttnConfig):
    return LinearMixFn.apply(q, k, v, u, feat, cfg)


# ---------------------------------------------------------------- scoring (K1)

@dataclass(frozen=True)
class ScoringConfig:
    """ScoringParams (proj/include/sparsek/selection.hpp:19-27) minus w_score."""
    slope_eps: float = 0.01
    slope_enabled: bool = True
    norm_mode: str = "timestep_norm"      # "timestep_norm" | "none"
    slope_order: str = "norm_then_slope"  # "norm_then_slope" | "slope_then_norm"
    chunk_len: int = 0                    # backward: norm pullback kept inside each chunk

    def c(self):
        return Scoring(int(self.norm_mode == "timestep_norm"),
                       int(self.slope_order == "norm_then_slope"), int(bool(self.slope_enabled)),
                       int(self.chunk_len), float(self.slope_eps))


@_on_device
def score_fwd(x: torch.Tensor, w: torch.Tensor, sc: ScoringConfig):
    """x [B, L, D] -> (raw, u, mean, sdev) float64 [B, L]."""
    if x.dim() != 3:
        raise _lib.ShapeError("score: x must be [B, L, D]")
    B, L, D = x.shape
    if w.shape != (D,):
        raise _lib.ShapeError("score_tokens: x.cols != w_score length")
    x = x.contiguous()
    w = w.to(torch.float64).contiguous()
    raw, u, mean, sdev = (torch.empty((B, L), dtype=torch.float64, device=x.device)
                          for _ in range(4))
    check(_lib.load().skb_score_fwd(B, L, D, _DT[x.dtype], x.data_ptr(), w.data_ptr(), sc.c(),
                                    raw.data_ptr(), u.data_ptr(), mean.data_ptr(), sdev.data_ptr(),
                                    _stream()))
    return raw, u, mean, sdev


@_on_device
def score_continue(x: torch.Tensor, w: torch.Tensor, sc: ScoringConfig, state: torch.Tensor):
    """Incremental scoring (score_tokens with a carried TimestepNormState,
    proj/src/selection.cpp:22-31): x [B, n, D] continues ``state`` (float64
    [B, 3] = count, mean, m2; updated in place). Returns (raw, u) [B, n]."""
    if x.dim() != 3:
        raise _lib.ShapeError("score: x must be [B, L, D]")
    B, n, D = x.shape
    if w.shape != (D,):
        raise _lib.ShapeError("score_tokens: x.cols != w_score length")
    if state.shape != (B, 3) or state.dtype != torch.float64 or not state.is_contiguous():
        raise _lib.ArgumentError("score_continue: state must be a contiguous float64 [B, 3]")
    x = x.contiguous()
    w = w.to(torch.float64).contiguous()
    raw, u = (torch.empty((B, n), dtype=torch.float64, device=x.device) for _ in range(2))
    check(_lib.load().skb_score_continue(B, n, D, _DT[x.dtype], x.data_ptr(), w.data_ptr(), sc.c(),
                                         state.data_ptr(), raw.data_ptr(), u.data_ptr(),
                                         _stream()))
    return raw, u


@_on_device
def score_bwd(x, w, sc: ScoringConfig, gu, raw, mean, sdev, dx=None, want_dw=True):
    B, L, D = x.shape
    graw = torch.empty((B, L), dtype=torch.float64, device=x.device)
    dw = torch.empty((D,), dtype=torch.float64, device=x.device) if want_dw else None
    check(_lib.load().skb_score_bwd(B, L, D, _DT[x.dtype], x.data_ptr(),
                                    w.to(torch.float64).contiguous().data_ptr(), sc.c(),
                                    gu.contiguous().data_ptr(), raw.data_ptr(), mean.data_ptr(),
                                    sdev.data_ptr(), graw.data_ptr(), _ptr(dw), _ptr(dx), _stream()))
    return graw, dw


class ScoreFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, sc: ScoringConfig):
        raw, u, mean, sdev = score_fwd(x, w, sc)
        ctx.save_for_backward(x, w, raw, mean, sdev)
        ctx.sc = sc
        return u

    @staticmethod
    def backward(ctx, gu):
        x, w, raw, mean, sdev = ctx.saved_tensors
        graw, dw = score_bwd(x, w, ctx.sc, gu.contiguous(), raw, mean, sdev)
        dx = (graw.unsqueeze(-1) * w.to(torch.float64)).to(x.dtype)
        return dx, dw.to(w.dtype), None


def score_tokens(x, w, sc: ScoringConfig):
    return ScoreFn.apply(x, w, sc)


def proj_supported(x, w):
    """The fused projection GEMM (skb_proj_score) covers bf16 with d_model a multiple of 256."""
    D = x.shape[-1]
    return (x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and D % 256 == 0 and x.is_cuda
            and w.shape == (D, D))


@_on_device
def proj_score(x, wq, wk, wv, w_score, sc: ScoringConfig):
    """forward_chunk's front (proj/src/cache.cpp:204-228) in one launch chain:
    q|k|v = x W* (hand-written tcgen05 GEMM) and, when w_score is given, the
    score (raw, u, mean, sdev) formed from the same x tiles (raw bit-identical
    to score_fwd). x [B, L, D] bf16; W* [D, D] bf16. Returns q, k, v [B, L, D]
    and the four float64 [B, L] score arrays (None without w_score)."""
    B, L, D = x.shape
    for w in (wq, wk, wv):
        if w.shape != (D, D) or w.dtype != torch.bfloat16:
            raise _lib.ShapeError("forward_chunk: projection shapes must be d_model x d_model")
    x = x.contiguous()
    wq, wk, wv = wq.contiguous(), wk.contiguous(), wv.contiguous()
    q, k, v = (torch.empty((B, L, D), dtype=torch.bfloat16, device=x.device) for _ in range(3))
    if w_score is not None:
        wsd = w_score.to(torch.float64).contiguous()
        raw, u, mean, sdev = (torch.empty((B, L), dtype=torch.float64, device=x.device) for _ in range(4))
        check(_lib.load().skb_proj_score(B, L, D, x.data_ptr(), wq.data_ptr(), wk.data_ptr(), wv.data_ptr(),
                                         wsd.data_ptr(), sc.c(), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         raw.data_ptr(), u.data_ptr(), mean.data_ptr(), sdev.data_ptr(),
                                         _stream()))
        return q, k, v, raw, u, mean, sdev
    check(_lib.load().skb_proj_score(B, L, D, x.data_ptr(), wq.data_ptr(), wk.data_ptr(), wv.data_ptr(), None,
                                     None, q.data_ptr(), k.data_ptr(), v.data_ptr(), None, None, None, None,
                                     _stream()))
    return q, k, v, None, None, None, None


class ProjScoreFn(torch.autograd.Function):
    """(x, Wq, Wk, Wv, w_score) -> (q, k, v, u) through the fused GEMM; the
    backward is the reference's dW = x^T d*, dx = sum d* W*^T (cuBLAS,
    proj/src/attention.cpp:551-573) plus the score pullback (skb_score_bwd)."""

    @staticmethod
    def forward(ctx, x, wq, wk, wv, w_score, sc: ScoringConfig):
        q, k, v, raw, u, mean, sdev = proj_score(x, wq, wk, wv, w_score, sc)
        ctx.save_for_backward(x, wq, wk, wv, w_score, raw, mean, sdev)
        ctx.sc = sc
        return q, k, v, u

    @staticmethod
    def backward(ctx, gq, gk, gv, gu):
        x, wq, wk, wv, w_score, raw, mean, sdev = ctx.saved_tensors
        B, L, D = x.shape
        x2 = x.reshape(B * L, D)
        gs = [torch.zeros_like(x) if g is None else g.contiguous() for g in (gq, gk, gv)]
        dx = gs[0] @ wq.t() + gs[1] @ wk.t() + gs[2] @ wv.t()
        dws = [x2.t() @ g.reshape(B * L, D) for g in gs]
        dwsc = None
        if w_score is not None and gu is not None:
            graw, dw = score_bwd(x, w_score, ctx.sc, gu.contiguous(), raw, mean, sdev)
            dx = dx + (graw.unsqueeze(-1) * w_score.to(torch.float64)).to(x.dtype)
            dwsc = dw.to(w_score.dtype)
        return dx, dws[0], dws[1], dws[2], dwsc, None


# ---------------------------------------------------------------- operator

@_on_device
def sparsek_rows(z: torch.Tensor, k: float):
    """Batched SparseK projection of the rows of z [n, m] (float64, CUDA)."""
    if z.dim() != 2 or z.dtype != torch.float64 or not z.is_cuda:
        raise _lib.ArgumentError("z must be a CUDA float64 [n, m] tensor")
    z = z.contiguous()
    n, m = z.shape
    p = torch.empty_like(z)
    tau = torch.empty(n, dtype=torch.float64, device=z.device)
    uc = torch.empty(n, dtype=torch.int64, device=z.device)
    wc = torch.empty(n, dtype=torch.int64, device=z.device)
    fl = torch.empty(n, dtype=torch.int32, device=z.device)
    check(_lib.load().skb_sparsek(n, m, z.data_ptr(), float(k), p.data_ptr(), tau.data_ptr(),
                                  uc.data_ptr(), wc.data_ptr(), fl.data_ptr(), _stream()))
    return p, tau, uc, wc, fl


@_on_device
def sparsek_jvp_rows(z: torch.Tensor, k: float, v: torch.Tensor):
    z = z.contiguous()
    v = v.to(torch.float64).contiguous()
    n, m = z.shape
    out = torch.empty_like(z)
    check(_lib.load().skb_sparsek_jvp(n, m, z.data_ptr(), float(k), v.data_ptr(), out.data_ptr(),
                                      _stream()))
    return out


@_on_device
def topk_hard_rows(z: torch.Tensor, k: int):
    z = z.contiguous()
    n, m = z.shape
    out = torch.empty_like(z)
    check(_lib.load().skb_topk_hard(n, m, z.data_ptr(), int(k), out.data_ptr(), _stream()))
    return out


# ---------------------------------------------------------------- decode (K5)

def _cache_dev(fn):
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **kw):
        with torch.cuda.device(self.device):
            return fn(self, *a, **kw)

    return wrapped


class DecodeCache:
    """Constant-(floor(k)+w) KV cache for generation over skb_cache_*:
    SparseKvCache + generate_step (proj/include/sparsek/cache.hpp:21-102,
    proj/src/cache.cpp:570-577) at the q/k/v/u level for a batch of B
    sequences. ``step`` consumes one new position per sequence (q/k/v
    [B, H, p], u float64 [B]) and returns o [B, H, p]; ``prefill`` appends a
    prompt (k/v [B, n, H, p], u [B, n]) without attending."""

    def __init__(self, batch, heads, head_dim, cfg: AttnConfig, max_len, dtype=torch.bfloat16,
                 device=None):
        import ctypes

        self.B, self.H, self.p = int(batch), int(heads), int(head_dim)
        self.cfg, self.dtype, self.max_len = cfg, dtype, int(max_len)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._desc = make_desc(self.B, self.max_len, self.H, self.p, cfg, dtype)
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(_lib.load().skb_cache_create(self._desc, ctypes.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().skb_cache_destroy(h)
            except Exception:
                pass
            self._h = None

    def _chk(self, t, shape, dtype, name):
        if tuple(t.shape) != tuple(shape):
            raise _lib.ShapeError(f"cache: {name} must be {tuple(shape)}, got {tuple(t.shape)}")
        if t.dtype != dtype or not t.is_cuda:
            raise _lib.ArgumentError(f"cache: {name} must be a CUDA {dtype} tensor")
        return t.contiguous()

    @_cache_dev
    def step(self, q, k, v, u, out=None):
        shp = (self.B, self.H, self.p)
        q, k, v = (self._chk(t, shp, self.dtype, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
        u = self._chk(u, (self.B,), torch.float64, "u")
        o = torch.empty_like(q) if out is None else out
        check(_lib.load().skb_cache_step(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         u.data_ptr(), o.data_ptr(), _stream()))
        return o

    @_cache_dev
    def prefill(self, k, v, u):
        n = k.shape[1]
        shp = (self.B, n, self.H, self.p)
        k, v = (self._chk(t, shp, self.dtype, nm) for t, nm in ((k, "k"), (v, "v")))
        u = self._chk(u, (self.B, n), torch.float64, "u")
        check(_lib.load().skb_cache_prefill(self._h, k.data_ptr(), v.data_ptr(), u.data_ptr(), n,
                                            _stream()))

    @_cache_dev
    def linmix_prefill(self, v, phk):
        """Linear mix (cfg.linear_mix): after prefill(k, v, u), record phi(k) of the
        retained rows and add the prompt to the prefix state (phk float64 [B, n, H, p])."""
        n = v.shape[1]
        v = self._chk(v, (self.B, n, self.H, self.p), self.dtype, "v")
        phk = self._chk(phk, (self.B, n, self.H, self.p), torch.float64, "phk")
        check(_lib.load().skb_cache_linmix_prefill(self._h, v.data_ptr(), phk.data_ptr(), n, _stream()))

    @_cache_dev
    def linmix_step(self, q, k, v, u, phq, phk, out=None):
        """One position of the linear-mix cache: returns the mixture readout o [B, H, p]."""
        shp = (self.B, self.H, self.p)
        q, k, v = (self._chk(t, shp, self.dtype, n) for t, n in ((q, "q"), (k, "k"), (v, "v")))
        phq, phk = (self._chk(t, shp, torch.float64, n) for t, n in ((phq, "phq"), (phk, "phk")))
        u = self._chk(u, (self.B,), torch.float64, "u")
        o = torch.empty_like(q) if out is None else out
        check(_lib.load().skb_cache_linmix_step(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), u.data_ptr(),
                                                phq.data_ptr(), phk.data_ptr(), o.data_ptr(), _stream()))
        return o

    @_cache_dev
    def snapshot(self, b=0, norm_state=None):
        """SparseKvCache::serialize payload of sequence b (proj/src/cache.cpp:416-475);
        norm_state = (count, mean, m2) of the scoring that fed this cache."""
        import ctypes

        ns = None if norm_state is None else (ctypes.c_double * 3)(*[float(x) for x in norm_state])
        n = ctypes.c_size_t(0)
        check(_lib.load().skb_cache_snapshot(self._h, int(b), ns, None, ctypes.byref(n), _stream()))
        buf = (ctypes.c_uint8 * n.value)()
        check(_lib.load().skb_cache_snapshot(self._h, int(b), ns, buf, ctypes.byref(n), _stream()))
        return bytes(buf[: n.value])

    @_cache_dev
    def restore(self, blob, b=0):
        """SparseKvCache::deserialize (proj/src/cache.cpp:477-545) into sequence b;
        returns the snapshot's norm state (count, mean, m2)."""
        import ctypes

        ns = (ctypes.c_double * 3)()
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(_lib.load().skb_cache_restore(self._h, int(b), buf, len(blob), ns, _stream()))
        return tuple(ns)

    @_cache_dev
    def state(self, b=0):
        """{positions (selected asc, then window asc), tau, seen, peak}."""
        import ctypes

        import numpy as np

        pos = np.zeros(max(1, int(math.floor(self.cfg.k)) + self.cfg.window + 1), np.int32)
        cnt, seen, peak = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        tau = ctypes.c_double()
        check(_lib.load().skb_cache_state(self._h, int(b), pos.ctypes.data, ctypes.byref(cnt),
                                          ctypes.byref(tau), ctypes.byref(seen), ctypes.byref(peak),
                                          _stream()))
        return {"positions": pos[: cnt.value].astype(np.int64), "tau": tau.value,
                "seen": seen.value, "peak": peak.value}
