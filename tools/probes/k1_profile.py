"""Per-kernel device times of one K1 score_fwd at cfg3's x shape (torch profiler / CUPTI)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
B, L, D = 2, 16384, 4096
x = torch.randn((B, L, D), device=dev).to(torch.bfloat16)
w = torch.randn((D,), device=dev, dtype=torch.float64) / math.sqrt(D)
sc = ops.ScoringConfig()
for _ in range(2):
    ops.score_fwd(x, w, sc)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ops.score_fwd(x, w, sc)
    torch.cuda.synchronize()
for ev in prof.events():
    if ev.device_type is not None and "CUDA" in str(ev.device_type):
        print(f"{ev.name[:90]:90s} {ev.device_time_total if hasattr(ev, 'device_time_total') else ev.cuda_time_total:10.1f} us")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
