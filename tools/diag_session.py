"""Diagnostics: where a float64 DecodeSession departs from the reference decode."""
import numpy as np
import torch

from oracle.oracle import Oracle, Reference, ref_cfg
from paper_2406_16747_b200 import DecodeSession, ops

L, D, H, k, w, km, mm, prompt = 80, 64, 4, 6.0, 0, "soft", "soft", 0
rng = np.random.default_rng(L + D)
x = rng.normal(size=(L, D))
ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
wsc = rng.normal(size=D)
ref = Reference()
y_ref, peak = ref.decode(x, *ws, wsc, ref_cfg(k, w, heads=H, key_mode=km, mask_mode=mm), prompt)
tape, _ = ref.attention(x, *ws, wsc, ref_cfg(k, w, heads=H, key_mode=km, mask_mode=mm))
print("batch ref vs decode ref", np.abs(tape.y - y_ref).max())
d = torch.device("cuda")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
q = (t(x) @ t(ws[0])).cpu().numpy()
print("q vs numpy", np.abs(q - x @ ws[0]).max(), "vs tape.q", np.abs(q - tape.q).max())
cfg = ops.AttnConfig(k=k, window=w, key_mode=km, mask_mode=mm)
s = DecodeSession(*(t(a) for a in ws), t(wsc), cfg, H, batch=1, max_len=L)
ys = [s.step(t(x)[i][None])[0] for i in range(L)]
y = torch.stack(ys).cpu().numpy()
err = np.abs(y - y_ref).max(1)
print("row err", np.array2string(err, precision=2))
st = torch.zeros((1, 3), dtype=torch.float64, device=d)
_, u = ops.score_continue(t(x)[None], t(wsc), ops.ScoringConfig(), st)
print("u vs tape.u", np.abs(u[0].cpu().numpy() - tape.u).max())
