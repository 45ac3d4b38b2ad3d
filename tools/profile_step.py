"""Run the bench workload for a few steps (for ncu captures): python tools/profile_step.py [steps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_16747_b200 import ops  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scores = sys.argv[2] if len(sys.argv) > 2 else "recency"
dev = torch.device("cuda", 0)
C = bench.CFG
cfg = ops.AttnConfig(k=C["k"], window=C["w"])
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, scores)
ws = ops.bwd_workspace(q, cfg)
for _ in range(steps):
    sel = ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
    o, lse, _ = ops.attn_fwd(q, k, v, u, cfg, sel=sel)
    ops.attn_bwd(q, k, v, o, do, lse, u, sel, cfg, ws=ws)
torch.cuda.synchronize()
print("ok")
