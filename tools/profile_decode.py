"""A few decode steps at cfg4 for ncu: python tools/profile_decode.py [steps] [ctx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device("cuda", 0)
B, H, d = 64, 32, 128
cache = ops.DecodeCache(B, H, d, ops.AttnConfig(k=1024.0, window=512), max_len=ctx + steps + 4)
g = torch.Generator(device=dev)
g.manual_seed(1)
kh = torch.randn((B, ctx, H, d), generator=g, device=dev).to(torch.bfloat16)
uh = torch.randn((B, ctx), generator=g, device=dev, dtype=torch.float64) + 0.01 * torch.arange(1, ctx + 1, device=dev)
cache.prefill(kh, kh, uh)
q = torch.randn((B, H, d), generator=g, device=dev).to(torch.bfloat16)
u = torch.randn((B,), generator=g, device=dev, dtype=torch.float64) + 0.01 * ctx
for _ in range(steps):
    cache.step(q, q, q, u)
torch.cuda.synchronize()
print("ok")
