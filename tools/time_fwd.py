import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2406_16747_b200 import ops
dev = torch.device("cuda", 0)
C = bench.CFG
cfg = ops.AttnConfig(k=C["k"], window=C["w"])
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, sys.argv[1] if len(sys.argv) > 1 else "recency")
sel = ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
for _ in range(3): ops.attn_fwd(q, k, v, u, cfg, sel=sel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ops.attn_fwd(q, k, v, u, cfg, sel=sel)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("SKB_LIB_PATH", "default"), "fwd ms", e0.elapsed_time(e1) / 10)
