"""Tensor-core path vs the f32 gather path with the persistent grids capped
(SKB_MAX_CTAS set by the caller), so every CTA walks many work items and every
ring wraps around many times. Prints one line per case; exits 1 on a mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
dev = torch.device("cuda", 0)
CASES = [  # L, H, D, k, w, kind, chunk_len
    (700, 2, 64, 100.5, 40, "recency", 0),
    (1500, 2, 128, 200.0, 100, "iid", 0),
] if small else [
    (2048, 3, 128, 300.5, 200, "recency", 0),
    (2500, 2, 64, 120.0, 64, "iid", 0),
    (3000, 2, 128, 256.0, 300, "iid", 512),
    (1777, 2, 128, 90.5, 33, "recency", 0),
    (2300, 2, 128, 150.0, 128, "mixed", 0),  # one dense, one sparse sequence: both backward paths at once
    (1900, 2, 64, 120.5, 96, "mixed", 0),
]
bad = 0
for L, H, D, k, w, kind, chunk in CASES:
    g = torch.Generator(device=dev)
    g.manual_seed(L + D)
    q, kk, v, do = (torch.randn((2, L, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    u = torch.randn((2, L), generator=g, device=dev, dtype=torch.float64)
    if kind == "recency":
        u += 0.01 * torch.arange(L, device=dev, dtype=torch.float64)
    elif kind == "mixed":
        u[0] += 0.01 * torch.arange(L, device=dev, dtype=torch.float64)
    res = {}
    for fg in (False, True):
        cfg = ops.AttnConfig(k=k, window=w, chunk_len=chunk, force_gather=fg)
        cast = (lambda t: t.float().contiguous()) if fg else (lambda t: t)
        o, lse, sel = ops.attn_fwd(cast(q), cast(kk), cast(v), u, cfg)
        res[fg] = (o,) + tuple(ops.attn_bwd(cast(q), cast(kk), cast(v), o, cast(do), lse, u, sel, cfg))
    torch.cuda.synchronize()
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))
    errs = {nm: rel(a, b) for nm, a, b in zip(("o", "dq", "dk", "dv", "du"), res[False], res[True])}
    ok = all(e < 2e-2 for nm, e in errs.items())
    bad += not ok
    print(("ok  " if ok else "BAD ") + str((L, H, D, k, w, kind, chunk)) + " " +
          " ".join(f"{nm}={e:.2e}" for nm, e in errs.items()), flush=True)
sys.exit(1 if bad else 0)
