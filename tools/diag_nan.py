"""Locate non-finite / mismatching dK rows of the tensor-core backward vs the gather path."""
import sys

import torch

from paper_2406_16747_b200 import ops

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cuda = torch.device("cuda")
B, L, H, p, k, w = 1, 2048, 2, 128, 300.0, 300
g = torch.Generator(device=cuda)
g.manual_seed(chunk)
q, kk, v, do = (torch.randn((B, L, H, p), generator=g, device=cuda).to(torch.bfloat16) for _ in range(4))
u = (torch.randn((B, L), generator=g, device=cuda, dtype=torch.float64)
     + 0.01 * torch.arange(1, L + 1, device=cuda, dtype=torch.float64))
res = {}
for fg in (False, True):
    cfg = ops.AttnConfig(k=k, window=w, chunk_len=chunk, force_gather=fg)
    cast = (lambda t: t.float().contiguous()) if fg else (lambda t: t)
    o, lse, sel = ops.attn_fwd(cast(q), cast(kk), cast(v), u, cfg)
    res[fg] = tuple(ops.attn_bwd(cast(q), cast(kk), cast(v), o, cast(do), lse, u, sel, cfg))
torch.cuda.synchronize()
for nm, i in (("dk", 1), ("dv", 2)):
    a, b = res[False][i].double(), res[True][i].double()
    bad = ~torch.isfinite(a)
    rows = bad.any(-1).any(-1)[0].nonzero().flatten().tolist()
    err = ((a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-9))[0]
    print(nm, "nonfinite rows", rows[:20], len(rows), "max row err", float(err[torch.isfinite(err)].max()),
          "worst rows", err.nan_to_num(1e9).max(-1).values.topk(5).indices.tolist())
