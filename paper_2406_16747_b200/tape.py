"""AttnTape and the tape-driven backward: the reference's training interface
(proj/include/sparsek/attention.hpp:47-91) over the B200 kernels.

``forward(x, params, scoring, cfg, tape)`` is sparsek_attention with a tape
(proj/src/attention.cpp:37-43 -> SparseKvCache::forward_chunk,
proj/src/cache.cpp:181-400); ``backward(tape, grad_out, params, scoring)`` is
sparsek_attention_backward (proj/src/attention.cpp:214-575) returning the
reference's AttnGrads fields. Everything stays on the device: the tape holds
the projections, the score recurrents, the selection products (leave
intervals and tau per push time) and the per-(query, head) log-sum-exp.

Memory: the reference tape keeps per query the attended list and gates,
O(L (k + w)); here the selection is O(L) (an interval per key), and
``queries`` rebuilds the reference's QueryRec view on demand (host side, for
inspection and parity tests). Softmax statistics: the reference keeps maxa
and denom per (query, head); the kernels keep lse = maxa + log(denom), and a
QueryRec reports maxa = lse, denom = 1 — the same softmax
exp(a - maxa) / denom for every logit a.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, ops


@dataclass
class AttnParams:
    """AttnParams<T> (proj/include/sparsek/attention.hpp:34-37): d x d, head h owns columns [h*p, (h+1)*p)."""
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor


@dataclass
class QueryRec:
    n_sel: int
    att: np.ndarray
    gate: np.ndarray
    maxa: np.ndarray
    denom: np.ndarray


@dataclass
class AttnTape:
    """AttnTape<T> (proj/include/sparsek/attention.hpp:47-68), device-resident."""
    x: torch.Tensor | None = None
    q: torch.Tensor | None = None
    k: torch.Tensor | None = None
    v: torch.Tensor | None = None
    head_concat: torch.Tensor | None = None
    raw: torch.Tensor | None = None
    u: torch.Tensor | None = None
    norm_mean: torch.Tensor | None = None
    norm_sdev: torch.Tensor | None = None
    lse: torch.Tensor | None = None
    selection: ops.Selection | None = None
    cfg: ops.AttnConfig | None = None
    heads: int = 1
    d_model: int = 0
    chunk_starts: list = field(default_factory=list)

    @property
    def tau_push(self) -> np.ndarray:
        """Stream tau after each score entered (push times 0 .. L-w-1), batch 0."""
        L, w = self.x.shape[1], self.cfg.window
        if self.selection is None or L <= w:
            return np.zeros(0)
        return self.selection.tau[0, : L - w].cpu().numpy()

    def queries(self, b: int = 0) -> list[QueryRec]:
        """The reference's per-query snapshot for sequence b: attended positions
        (selected ascending, then the window ascending), gates of the selected
        entries, and per-head softmax statistics."""
        L = self.x.shape[1]
        w = self.cfg.window
        kf = int(math.floor(self.cfg.k))
        u = self.u[b].cpu().numpy()
        lse = self.lse[b].cpu().numpy()  # [H, L]
        if self.selection is not None and kf >= 1:
            leave = self.selection.leave[b].cpu().numpy()
            tq = self.selection.tau_per_query()[b].cpu().numpy()
        else:
            leave, tq = None, np.full(L, -np.inf)
        out = []
        for i in range(L):
            t = i - w
            if leave is not None and t >= 0:
                js = np.arange(t + 1)
                sel = js[leave[: t + 1] > t]
            else:
                sel = np.zeros(0, np.int64)
            win = np.arange(max(0, i - w + 1), i + 1) if w > 0 else np.zeros(0, np.int64)
            if w == 0 and not np.any(sel == i):
                win = np.array([i])
            gate = np.clip(u[sel] - tq[i], 0.0, 1.0) if sel.size else np.zeros(0)
            out.append(QueryRec(int(sel.size), np.concatenate([sel, win]).astype(np.uint32), gate,
                                lse[:, i].copy(), np.ones(lse.shape[0])))
        return out


def _check_x(x, params: AttnParams, heads):
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if x.dim() != 3:
        raise _lib.ShapeError("forward_chunk: x must be [L, D] or [B, L, D]")
    D = x.shape[-1]
    for w in (params.wq, params.wk, params.wv, params.wo):
        if tuple(w.shape) != (D, D):
            raise _lib.ShapeError("forward_chunk: projection shapes must be d_model x d_model")
    if heads <= 0 or D % heads:
        raise _lib.ConfigError("attention: d_model must be a positive multiple of heads")
    return x


@torch.no_grad()
def forward(x: torch.Tensor, params: AttnParams, w_score: torch.Tensor | None,
            scoring: ops.ScoringConfig, cfg: ops.AttnConfig, heads: int,
            tape: AttnTape | None = None) -> torch.Tensor:
    """sparsek_attention<T> (proj/src/attention.cpp:37-43) on device tensors.
    x: [L, D] or [B, L, D]; returns y of the same shape. Fills `tape` when given."""
    squeeze = x.dim() == 2
    x = _check_x(x, params, heads).contiguous()
    B, L, D = x.shape
    p = D // heads
    q = (x @ params.wq).view(B, L, heads, p).contiguous()
    k = (x @ params.wk).view(B, L, heads, p).contiguous()
    v = (x @ params.wv).view(B, L, heads, p).contiguous()
    if cfg.k > 0.0:
        if w_score is None or tuple(w_score.shape) != (D,):
            raise _lib.ConfigError("attention: w_score length must equal d_model")
        raw, u, mean, sdev = ops.score_fwd(x, w_score, scoring)
    else:
        raw = u = mean = sdev = torch.zeros((B, L), dtype=torch.float64, device=x.device)
    o, lse, sel = ops.attn_fwd(q, k, v, u, cfg)
    hc = o.view(B, L, D)
    y = hc @ params.wo
    if tape is not None:
        tape.x, tape.q, tape.k, tape.v, tape.head_concat = x, q, k, v, o
        tape.raw, tape.u, tape.norm_mean, tape.norm_sdev = raw, u, mean, sdev
        tape.lse, tape.selection, tape.cfg = lse, sel, cfg
        tape.heads, tape.d_model = heads, D
        cl = cfg.chunk_len if cfg.chunk_len > 0 else L
        tape.chunk_starts = list(range(0, L, cl))
    return y[0] if squeeze else y


@torch.no_grad()
def backward(tape: AttnTape, grad_out: torch.Tensor, params: AttnParams, w_score: torch.Tensor | None,
             scoring: ops.ScoringConfig) -> dict:
    """sparsek_attention_backward (proj/src/attention.cpp:214-575): returns the
    AttnGrads fields {dx, dwq, dwk, dwv, dwo, dw_score} from a tape."""
    if tape.x is None:
        raise _lib.ArgumentError("sparsek_attention_backward: empty tape")
    x = tape.x
    B, L, D = x.shape
    g = grad_out.view(B, L, D).to(x.dtype).contiguous()
    xf = x.reshape(B * L, D)
    hc = tape.head_concat.reshape(B * L, D)
    dwo = hc.t() @ g.reshape(B * L, D)                                   # attention.cpp:236-247
    dhc = (g.reshape(B * L, D) @ params.wo.t()).view_as(tape.q).contiguous()
    dq, dk, dv, du = ops.attn_bwd(tape.q, tape.k, tape.v, tape.head_concat, dhc, tape.lse, tape.u,
                                  tape.selection, tape.cfg)
    dqf, dkf, dvf = (t.reshape(B * L, D) for t in (dq, dk, dv))
    dwq, dwk, dwv = xf.t() @ dqf, xf.t() @ dkf, xf.t() @ dvf          # attention.cpp:551-573
    dx = dqf @ params.wq.t() + dkf @ params.wk.t() + dvf @ params.wv.t()
    dw_score = None
    if tape.cfg.k > 0.0:
        sc = scoring if tape.cfg.chunk_len <= 0 else ops.ScoringConfig(
            slope_eps=scoring.slope_eps, slope_enabled=scoring.slope_enabled, norm_mode=scoring.norm_mode,
            slope_order=scoring.slope_order, chunk_len=int(tape.cfg.chunk_len))
        graw, dw_score = ops.score_bwd(x, w_score, sc, du, tape.raw, tape.norm_mean, tape.norm_sdev)
        dx = dx + (graw.reshape(B * L, 1) * w_score.to(torch.float64).view(1, D)).to(dx.dtype)  # :564
    else:
        dw_score = torch.zeros(D, dtype=torch.float64, device=x.device)
    return dict(dx=dx.view(B, L, D), dwq=dwq, dwk=dwk, dwv=dwv, dwo=dwo, dw_score=dw_score)
