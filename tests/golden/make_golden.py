"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
Each fixture is a core-level problem driven through the reference's own
sparsek_attention / sparsek_attention_backward with the identity-input trick
(x = I, W = Q/K/V, Wo = I; see oracle/oracle.py:core_problem_via_reference),
so the stored outputs are exactly the reference's.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference, core_problem_via_reference  # noqa: E402

CASES = [
    # name, H, p, k, w, key_mode, mask_mode, norm_mode, slope, seed
    ("core_hard_soft_none", 2, 32, 8.5, 8, "hard", "soft", "none", False, 11),
    ("core_soft_st_norm", 2, 32, 6.0, 5, "soft", "straight_through", "timestep_norm", True, 12),
    ("core_w0_k7", 4, 16, 7.0, 0, "hard", "soft", "timestep_norm", True, 13),
    ("core_ties", 2, 32, 4.0, 3, "hard", "soft", "none", False, 14),
]


def main():
    ref = Reference()
    for name, H, p, k, w, km, mm, nm, slope, seed in CASES:
        rng = np.random.default_rng(seed)
        L = H * p
        Q, K, V, dO = (rng.normal(size=(L, H, p)) for _ in range(4))
        if name == "core_ties":
            ws = 0.5 * rng.integers(-3, 4, size=L).astype(np.float64)  # heavy ties
        else:
            ws = rng.normal(size=L)
        tape, grads = core_problem_via_reference(ref, Q, K, V, ws, dO, kbudget=k, window=w,
                                                 key_mode=km, mask_mode=mm, norm_mode=nm,
                                                 slope_enabled=slope)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), H=H, p=p, k=k, w=w, key_mode=km, mask_mode=mm,
            norm_mode=nm, slope=slope, Q=Q, K=K, V=V, dO=dO, w_score=ws, u=tape.u, raw=tape.raw,
            norm_mean=tape.norm_mean, norm_sdev=tape.norm_sdev, tau_push=tape.tau_push,
            n_sel=tape.n_sel, att_off=tape.att_off, att=tape.att, gate=tape.gate,
            head_concat=tape.head_concat, maxa=tape.maxa, denom=tape.denom, dq=grads["dwq"],
            dk=grads["dwk"], dv=grads["dwv"], dw_score=grads["dw_score"])
        print("wrote", name)


if __name__ == "__main__":
    main()
