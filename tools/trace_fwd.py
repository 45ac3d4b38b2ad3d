"""Per-tile pipeline timeline of one forward CTA (needs a -DSKB_TRACE build):
SKB_LIB_PATH=.../libsparsek_b200.so python tools/trace_fwd.py [recency|iid]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_16747_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
C = bench.CFG
cfg = ops.AttnConfig(k=C["k"], window=C["w"])
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, sys.argv[1] if len(sys.argv) > 1 else "recency")
sel = ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
for _ in range(3):
    ops.attn_fwd(q, k, v, u, cfg, sel=sel)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
_lib.load().skb_debug_trace(buf, 4096)
t = np.array(buf, dtype=np.int64)
roles = {0: "WG0", 1: "WG1", 2: "PROD", 3: "MMA"}
names = {0: {9: "wS", 0: "S", 1: "ld", 2: "max", 3: "exp", 4: "P"}, 1: {9: "wS", 0: "S", 1: "ld", 2: "max", 3: "exp", 4: "P"},
         2: {0: "it", 1: "Kgo", 2: "Kdone", 3: "Vgo", 4: "Vdone"}, 3: {8: "wK", 0: "K", 1: "QK", 2: "P0", 3: "P1"}}
t0 = min(x for x in t if x > 0)
for jt in range(16):
    row = []
    for r in range(4):
        for ev, nm in names[r].items():
            x = t[r * 256 + jt * 16 + ev]
            if x > 0:
                row.append(f"{roles[r]}.{nm}={x - t0}")
    if row:
        print(f"tile {jt:2d}: " + " ".join(row))
