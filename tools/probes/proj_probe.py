"""Step-by-step probe of the fused projection kernel (each step flushed)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

mode = sys.argv[1]
dev = torch.device("cuda", 0)
B, L, D = 1, 256, 256
x = torch.randn((B, L, D), device=dev).to(torch.bfloat16)
ws = [(torch.randn((D, D), device=dev) / 16).to(torch.bfloat16) for _ in range(3)]
wsc = torch.randn((D,), device=dev, dtype=torch.float64)
sc = ops.ScoringConfig()
t = time.time()
if mode == "noscore":
    q, k, v, *_ = ops.proj_score(x, *ws, None, sc)
elif mode == "none":
    q, k, v, *_ = ops.proj_score(x, *ws, wsc, ops.ScoringConfig(norm_mode="none"))
else:
    q, k, v, *_ = ops.proj_score(x, *ws, wsc, sc)
torch.cuda.synchronize()
err = ((q.float() - x.float() @ ws[0].float()).norm() / (x.float() @ ws[0].float()).norm()).item()
print(mode, "ok", time.time() - t, "err", err, flush=True)
