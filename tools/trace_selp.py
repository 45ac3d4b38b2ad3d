"""Timeline of items 6.. of one persistent selected-pass dK/dV CTA (-DSKB_TRACE -DSKB_TRACE_SEL)."""
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
buf = (ctypes.c_ulonglong * 8192)()
_lib.load().skb_debug_trace_bwd(buf, 8192)
tt = np.array(buf, dtype=np.int64)
for cta in (0, 1):
    t = tt[cta * 4096:(cta + 1) * 4096]
    if not (t > 0).any():
        continue
    print(f"== CTA {100 + cta}")
    names = {4: {9: "wS", 0: "S", 4: "PdS", 5: "accD", 6: "end"}, 6: {3: "fetched", 2: "KVgo", 1: "Qgo"},
             7: {4: "KV", 0: "Q", 1: "SdP", 2: "PdS"}}
    names[5] = names[4]
    roles = {4: "WG0", 5: "WG1", 6: "PROD", 7: "MMA"}
    t0 = min(x for x in np.concatenate([tt[4 * 512:8 * 512], tt[4096 + 4 * 512:4096 + 8 * 512]]) if x > 0)
    for jt in range(32):
        row = []
        for r in (7, 4, 5, 6):
            for ev, nm in names[r].items():
                x = t[(r * 512 + jt * 16 + ev) & 4095]
                if x > 0:
                    row.append(f"{roles[r]}.{nm}={x - t0}")
        if row:
            print(f"g{jt:2d}: " + " ".join(row))
