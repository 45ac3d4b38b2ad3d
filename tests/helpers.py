"""Shared test helpers: drive the GPU core path from numpy and rebuild the
reference's per-query snapshot (att lists, gates) from the device products."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(path):
    z = np.load(path, allow_pickle=False)
    return {k: (z[k].item() if z[k].ndim == 0 else z[k]) for k in z.files}


def sel_lists_from_leave(leave, L, w):
    """Sel_i (ascending) per query from leave intervals: j <= t < leave_j, t = i - w."""
    T = max(0, L - w)
    out = []
    for i in range(L):
        t = i - w
        if t < 0:
            out.append(np.zeros(0, np.int64))
            continue
        js = np.arange(0, t + 1)
        out.append(js[leave[: t + 1] > t])
    return out


def run_core_gpu(Q, K, V, u, dO, *, k, w, key_mode="hard", mask_mode="soft", dtype="f64",
                 force_gather=False, device="cuda"):
    """Q/K/V/dO: [L, H, p] or [B, L, H, p] numpy; u [L] or [B, L]. Returns dict of numpy."""
    import torch

    from paper_2406_16747_b200 import ops

    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    squeeze = Q.ndim == 3
    if squeeze:
        Q, K, V, dO, u = Q[None], K[None], V[None], dO[None] if dO is not None else None, u[None]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device).to(tdt)
    q, kk, v = t(Q), t(K), t(V)
    ut = torch.from_numpy(np.ascontiguousarray(u, np.float64)).to(device)
    cfg = ops.AttnConfig(k=float(k), window=int(w), key_mode=key_mode, mask_mode=mask_mode,
                         force_gather=force_gather)
    o, lse, sel = ops.attn_fwd(q, kk, v, ut, cfg)
    res = dict(o=o.double().cpu().numpy(), lse=lse.cpu().numpy(),
               leave=sel.leave.cpu().numpy(), tau=sel.tau.cpu().numpy(),
               nfrac=sel.nfrac.cpu().numpy(), tau_q=sel.tau_per_query().cpu().numpy())
    if dO is not None:
        dq, dk, dv, du = ops.attn_bwd(q, kk, v, o, t(dO), lse, ut, sel, cfg)
        res.update(dq=dq.double().cpu().numpy(), dk=dk.double().cpu().numpy(),
                   dv=dv.double().cpu().numpy(), du=du.cpu().numpy())
    torch.cuda.synchronize()
    if squeeze:
        for key in list(res):
            res[key] = res[key][0]
    return res


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
