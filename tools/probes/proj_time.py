"""Time the fused projection front vs cuBLAS at cfg3's x shape (for ncu: argv[1] = fused|library|both)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
dev = torch.device("cuda", 0)
B, L, D = 2, 16384, 4096
x = torch.randn((B, L, D), device=dev).to(torch.bfloat16)
ws = [(torch.randn((D, D), device=dev) / math.sqrt(D)).to(torch.bfloat16) for _ in range(3)]
wsc = torch.randn((D,), device=dev, dtype=torch.float64) / math.sqrt(D)
sc = ops.ScoringConfig()
for _ in range(3):
    if which in ("fused", "both"):
        ops.proj_score(x, *ws, wsc, sc)
        ops.proj_score(x, *ws, None, sc)
    if which in ("library", "both"):
        for w in ws:
            x @ w
torch.cuda.synchronize()
print("ok")
