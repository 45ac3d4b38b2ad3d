"""Multi-GPU plumbing for the SparseK path: (batch, head) sharding over
``torch.distributed`` ranks, one process per GPU.

Units are independent (b, h) pairs: attention forward
and backward for a unit read only Q/K/V[b, :, h] and the selection of
sequence b, which every rank recomputes from u[b, :] (L floats) - no
collective on the data path. The one real exchange is the selection pullback:
the gate gradient is summed over heads before the JVP
(proj/src/attention.cpp:263,295,313), and the JVP is linear in those sums, so
each rank's du (from its heads) is a partial that is all-reduced (sum) among
the ranks sharing a sequence. Gathering outputs/gradients to one owner is an
optional all-gather (``gather_heads``).

The host logic here is backend-agnostic (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous head range [h0, h1) of `rank` (as even as possible)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("head_shard: bad world/rank")
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def unit_shard(B: int, H: int, world: int, rank: int) -> list[tuple[int, int, int]]:
    """The (b, h0, h1) blocks of `rank` when the B*H units are split into
    `world` contiguous ranges (b-major): e.g. cfg3 (B=2, H=32) over 8 GPUs gives
    every GPU 8 heads of one sequence."""
    units = B * H
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    out = []
    u = u0
    while u < u1:
        b, h = divmod(u, H)
        h1 = min(H, h + (u1 - u))
        out.append((b, h, h1))
        u += h1 - h
    return out


def seq_ranks(B: int, H: int, world: int) -> dict[int, list[int]]:
    """Sequence b -> the ranks whose unit_shard blocks hold heads of b (the
    ranks that all-reduce du[b])."""
    out: dict[int, list[int]] = {}
    for r in range(world):
        for b, _, _ in unit_shard(B, H, world, r):
            out.setdefault(b, []).append(r)
    return out


def allreduce_du(du: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank selection-pullback partials du[b, :] in place."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(du, op=dist.ReduceOp.SUM, group=group)
    return du


def gather_heads(x_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather head shards [B, L, H_local, p] -> [B, L, H, p] (equal shards)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return x_local
    parts = [torch.empty_like(x_local) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, x_local.contiguous(), group=group)
    return torch.cat(parts, dim=2)


class HeadParallelSparseK(torch.autograd.Function):
    """SparseK attention on this rank's heads; du all-reduced in backward.
    q/k/v: [B, L, H_local, p] device tensors of this rank; u: [B, L] float64
    (replicated)."""

    @staticmethod
    def forward(ctx, q, k, v, u, cfg, group=None):
        from . import ops

        q, k, v, u = q.contiguous(), k.contiguous(), v.contiguous(), u.contiguous()
        o, lse, sel = ops.attn_fwd(q, k, v, u, cfg)
        ctx.save_for_backward(q, k, v, o, lse, u)
        ctx.sel, ctx.cfg, ctx.group = sel, cfg, group
        return o

    @staticmethod
    def backward(ctx, do):
        from . import ops

        q, k, v, o, lse, u = ctx.saved_tensors
        dq, dk, dv, du = ops.attn_bwd(q, k, v, o, do, lse, u, ctx.sel, ctx.cfg)
        allreduce_du(du, ctx.group)
        return dq, dk, dv, du, None, None


def head_parallel_attention(q, k, v, u, cfg, group=None):
    return HeadParallelSparseK.apply(q, k, v, u, cfg, group)
