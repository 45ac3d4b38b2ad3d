"""Selection (K2) alone at a config, for launch lists: python tools/probes/select_profile.py B L k w [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

B, L, k, w = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
dev = torch.device("cuda", 0)
u = torch.randn((B, L), device=dev, dtype=torch.float64) + 0.01 * torch.arange(1, L + 1, device=dev)
cfg = ops.AttnConfig(k=k, window=w)
for _ in range(reps):
    ops.select(u, cfg, heads=8, head_dim=128, dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok")
