"""Timeline of items 6.. of one persistent dQ CTA (-DSKB_TRACE -DSKB_TRACE_DQP build)."""
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
o, lse, _ = ops.attn_fwd(q, k, v, u, cfg, sel=sel)
for _ in range(2):
    ops.attn_bwd(q, k, v, o, do, lse, u, sel, cfg)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
_lib.load().skb_debug_trace_bwd(buf, 4096)
t = np.array(buf, dtype=np.int64)
names = {0: {9: "wS", 0: "S", 4: "dS", 5: "last", 6: "dqD", 7: "dqOut"}, 2: {2: "KVgo"},
         3: {3: "Qfull", 4: "dOfull", 0: "KV", 1: "SdP", 2: "DS"}}
names[1] = names[0]
roles = {0: "WG0", 1: "WG1", 2: "PROD", 3: "MMA"}
t0 = min(x for x in t[:4 * 512] if x > 0)
for jt in range(32):
    row = []
    for r in (3, 0, 1, 2):
        for ev, nm in names[r].items():
            x = t[(r * 512 + jt * 16 + ev) & 4095]
            if x > 0:
                row.append(f"{roles[r]}.{nm}={x - t0}")
    if row:
        print(f"J{jt:2d}: " + " ".join(row))
