"""Writes the forward/backward outputs of a fixed problem to a .pt file (used to
check that the persistent grid size never changes a single bit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for L, H, D, k, w, kind in ((4000, 4, 128, 300.5, 200, "recency"), (3000, 3, 64, 150.0, 64, "iid")):
    g = torch.Generator(device=dev)
    g.manual_seed(L)
    q, kk, v, do = (torch.randn((2, L, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    u = torch.randn((2, L), generator=g, device=dev, dtype=torch.float64)
    if kind == "recency":
        u += 0.01 * torch.arange(L, device=dev, dtype=torch.float64)
    cfg = ops.AttnConfig(k=k, window=w)
    o, lse, sel = ops.attn_fwd(q, kk, v, u, cfg)
    dq, dk, dv, du = ops.attn_bwd(q, kk, v, o, do, lse, u, sel, cfg)
    out[kind] = [t.cpu() for t in (o, lse, dq, dk, dv)]
torch.save(out, sys.argv[1])
