"""Phase clocks of sequence 0's last tau chunk, including the segmented second pass (-DSKB_TRACE_TAU):
python tools/trace_tauseg.py [iid|recency]"""
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
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, sys.argv[1] if len(sys.argv) > 1 else "iid")
for _ in range(2):
    ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib = _lib.load()
lib.skb_debug_trace_tau.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.skb_debug_trace_tau(ctypes.cast(buf, ctypes.c_void_p), 16)
t = list(buf)
print("pass-1 band: theta", t[1] - t[0], "collect", t[2] - t[1])
print("segment: start->band sorted", t[8] - t[7], "band->last chunk", t[9] - t[8], "merge", t[10] - t[9],
      "prefix", t[4] - t[10], "solve", t[5] - t[4], "replay", t[6] - t[5], "total", t[6] - t[7])
