"""Timeline of tiles 12.. of CTA 100 in the 128-query unified pass (-DSKB_TRACE -DSKB_TRACE_KMAJ)."""
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
q, k, v, do, u = bench.make_inputs(torch, dev, 1234, "recency")
sel = ops.select(u, cfg, heads=C["H"], head_dim=C["d"], dtype=torch.bfloat16)
o, lse, _ = ops.attn_fwd(q, k, v, u, cfg, sel=sel)
for _ in range(2):
    ops.attn_bwd(q, k, v, o, do, lse, u, sel, cfg)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8192)()
_lib.load().skb_debug_trace_bwd(buf, 8192)
t = np.array(buf[:4096], dtype=np.int64)
names = {7: {0: "Q", 5: "R", 1: "S", 2: "accW", 6: "accI", 7: "R2", 3: "dP"},
         4: {9: "wS", 0: "Sld", 1: "P", 2: "PDE", 3: "dPw", 4: "dS"}}
names[5] = names[4]
roles = {4: "WG0", 5: "WG1", 7: "MMA"}
vals = [x for x in t[4 * 512:8 * 512] if x > 0]
t0 = min(vals)
for jt in range(24):
    row = []
    for r in (7, 4, 5):
        for ev, nm in names[r].items():
            x = t[(r * 512 + jt * 16 + ev) & 4095]
            if x > 0:
                row.append(f"{roles[r]}.{nm}={x - t0}")
    if row:
        print(f"g{jt:2d}: " + " ".join(row))
