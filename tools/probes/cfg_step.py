"""A few fwd+bwd steps at a config (for launch lists): python tools/probes/cfg_step.py B H L d k w [steps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2406_16747_b200 import ops  # noqa: E402

B, H, L, d = (int(x) for x in sys.argv[1:5])
k, w = float(sys.argv[5]), int(sys.argv[6])
steps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
dev = torch.device("cuda", 0)
q, kk, v, do = (torch.randn((B, L, H, d), device=dev).to(torch.bfloat16) for _ in range(4))
u = torch.randn((B, L), device=dev, dtype=torch.float64) + 0.01 * torch.arange(1, L + 1, device=dev)
cfg = ops.AttnConfig(k=k, window=w)
ws = ops.bwd_workspace(q, cfg)
for _ in range(steps):
    sel = ops.select(u, cfg, heads=H, head_dim=d, dtype=torch.bfloat16)
    o, lse, _ = ops.attn_fwd(q, kk, v, u, cfg, sel=sel)
    ops.attn_bwd(q, kk, v, o, do, lse, u, sel, cfg, ws=ws)
torch.cuda.synchronize()
print("ok")
