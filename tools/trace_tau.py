"""Phase clocks of the last tau chunk of sequence 0 (-DSKB_TRACE_TAU build): theta, band
collection, sort, prefix sums, exact solve, replay."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_16747_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
C = bench.CFG
cfg = ops.AttnConfig(k=C["k"], window=C["w"])
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, sys.argv[1] if len(sys.argv) > 1 else "recency")
for _ in range(2):
    ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib = _lib.load()
lib.skb_debug_trace_tau.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.skb_debug_trace_tau(ctypes.cast(buf, ctypes.c_void_p), 16)
t = list(buf)
names = ["start", "theta", "collect", "sort", "prefix", "solve", "replay"]
print(" ".join(f"{names[i]}=+{t[i] - t[i - 1]}" for i in range(1, 7)), "total", t[6] - t[0])
