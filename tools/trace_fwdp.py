"""Per-tile timeline of items 3.. of persistent forward CTA 100 (-DSKB_TRACE -DSKB_TRACE_FWDP build)."""
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
names = {3: {0: "K", 1: "S", 2: "pvV", 3: "P0", 4: "P1", 5: "PV"}, 0: {9: "wS", 0: "Sld", 4: "P"},
         2: {1: "Kgo", 3: "Vgo"}}
names[1] = names[0]
roles = {0: "WG0", 1: "WG1", 2: "PROD", 3: "MMA"}
t0 = min(x for x in t if x > 0)
for jt in range(16):
    row = []
    for r in (3, 0, 1, 2):
        for ev, nm in names[r].items():
            x = t[r * 256 + jt * 16 + ev]
            if x > 0:
                row.append(f"{roles[r]}.{nm}={x - t0}")
    if row:
        print(f"J{jt:2d}: " + " ".join(row))
