"""Print the observed relative errors of the core path against the oracle for
the parity-test cases (used to set and justify the test tolerances)."""
import json
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import rel_err, run_core_gpu  # noqa: E402
from tests.test_core_gpu import CASES, TC_CASES, _oracle_core, _scores  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

import torch  # noqa: E402

orc = Oracle()
rows = []
for cases, tag in ((CASES, "core"), (TC_CASES, "tc")):
    for case in cases:
        L, H, p, k, w, km, mm, kind = case
        for dtype in (("f32", "bf16") if tag == "core" else ("bf16",)):
            rng = np.random.default_rng(L * 7 + H if tag == "core" else L + 13 * H + p)
            Q, K, V, dO = (rng.normal(size=(L, H, p)) for _ in range(4))
            u = _scores(rng, L, kind)
            if dtype == "bf16":
                rnd = lambda a: torch.from_numpy(a).to(torch.bfloat16).double().numpy()
                Q, K, V, dO = rnd(Q), rnd(K), rnd(V), rnd(dO)
            sel, o, lse, dq, dk, dv, gu = _oracle_core(orc, Q, K, V, u, dO, k, w, km, mm)
            res = run_core_gpu(Q, K, V, u, dO, k=k, w=w, key_mode=km, mask_mode=mm, dtype=dtype)
            e = {n: rel_err(res[n], r) for n, r in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv))}
            e["du"] = rel_err(res["du"], gu) if np.abs(gu).max() > 0 else 0.0
            e["du_abs_over_scale"] = float(np.abs(res["du"] - gu).max() / max(np.abs(gu).max(), 1e-30))
            rows.append(dict(tag=tag, case=str(case), dtype=dtype, **e))
            print(json.dumps(rows[-1]), flush=True)
print("MAX", json.dumps({k: max(r[k] for r in rows) for k in ("o", "dq", "dk", "dv", "du")}))
for dt in ("f32", "bf16"):
    print("MAX", dt, json.dumps({k: max(r[k] for r in rows if r["dtype"] == dt) for k in ("o", "dq", "dk", "dv", "du")}))
