"""Fused projection front in three modes for a launch-metric A/B: plain GEMM, GEMM + raw (no norm), GEMM + full streaming score."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
B, L, D = 2, 16384, 4096
x = torch.randn((B, L, D), device=dev).to(torch.bfloat16)
ws = [(torch.randn((D, D), device=dev) / math.sqrt(D)).to(torch.bfloat16) for _ in range(3)]
wsc = torch.randn((D,), device=dev, dtype=torch.float64) / math.sqrt(D)
for _ in range(2):
    ops.proj_score(x, *ws, None, ops.ScoringConfig())
    ops.proj_score(x, *ws, wsc, ops.ScoringConfig(norm_mode="none"))
    ops.proj_score(x, *ws, wsc, ops.ScoringConfig())
torch.cuda.synchronize()
print("ok")
