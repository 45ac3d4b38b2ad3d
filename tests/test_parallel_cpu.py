"""CPU: the multi-rank host path (paper_2406_16747_b200.parallel) under gloo,
world_size 2. The per-rank compute is the C oracle (the GPU kernels need a
device); what is under test is the sharding and the du all-reduce: the
selection pullback is linear in the head-summed gate gradients, so the sum of
per-rank partials must equal the single-process result
(proj/src/attention.cpp:263,295,447-479)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_16747_b200.parallel import head_shard, unit_shard


def test_head_shard_covers_every_head_once():
    for H in (1, 5, 12, 32):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                h0, h1 = head_shard(H, world, r)
                seen += list(range(h0, h1))
            assert seen == list(range(H))


def test_unit_shard_cfg3_layout():
    # cfg3 over 8 GPUs: every GPU gets 8 heads of one sequence
    assert [unit_shard(2, 32, 8, r) for r in range(8)] == [
        [(0, 0, 8)], [(0, 8, 16)], [(0, 16, 24)], [(0, 24, 32)],
        [(1, 0, 8)], [(1, 8, 16)], [(1, 16, 24)], [(1, 24, 32)]]
    for B, H, world in ((3, 5, 4), (1, 7, 2), (2, 3, 6)):
        units = []
        for r in range(world):
            for b, h0, h1 in unit_shard(B, H, world, r):
                units += [(b, h) for h in range(h0, h1)]
        assert units == [(b, h) for b in range(B) for h in range(H)]


def test_seq_ranks_groups():
    from paper_2406_16747_b200.parallel import seq_ranks

    assert seq_ranks(2, 32, 1) == {0: [0], 1: [0]}
    assert seq_ranks(2, 32, 2) == {0: [0], 1: [1]}
    assert seq_ranks(2, 32, 4) == {0: [0, 1], 1: [2, 3]}
    assert seq_ranks(2, 32, 8) == {0: [0, 1, 2, 3], 1: [4, 5, 6, 7]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2406_16747_b200.parallel import allreduce_du, head_shard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(7)
    L, H, p, k, w = 160, 4, 8, 10.5, 6
    Q, K, V, dO = (rng.normal(size=(L, H, p)) for _ in range(4))
    u = rng.normal(size=L)
    orc = Oracle()
    sel = orc.select(u, k, w)
    h0, h1 = head_shard(H, world, rank)
    sl = slice(h0, h1)
    o, maxa, den = orc.attn_fwd(Q[:, sl], K[:, sl], V[:, sl], sel, kbudget=k, window=w)
    _, _, _, gu = orc.attn_bwd(Q[:, sl], K[:, sl], V[:, sl], dO[:, sl], u, sel, maxa, den,
                               kbudget=k, window=w)
    du = torch.from_numpy(gu.copy()).view(1, L)
    allreduce_du(du)
    if rank == 0:
        o_f, ma_f, de_f = orc.attn_fwd(Q, K, V, sel, kbudget=k, window=w)
        _, _, _, gu_full = orc.attn_bwd(Q, K, V, dO, u, sel, ma_f, de_f, kbudget=k, window=w)
        out["err"] = float(np.abs(du.numpy()[0] - gu_full).max() / max(np.abs(gu_full).max(), 1e-30))
    dist.barrier()
    dist.destroy_process_group()


def _run(rank, world, port, q):
    out = {}
    _worker(rank, world, port, out)
    if rank == 0:
        q.put(out["err"])


@pytest.mark.timeout(300)
def test_du_allreduce_over_head_shards_gloo():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    err = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert err < 1e-12, err
