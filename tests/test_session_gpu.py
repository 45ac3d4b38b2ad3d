"""GPU: x-level generation (DecodeSession) against the reference's own
SparseKvCache: forward_chunk on the prompt, then generate_step per row
(proj/src/cache.cpp:195-230,570-577), run by the C reference build
(oracle/_ref, ref_decode_run). The incremental score (skb_score_continue)
must reproduce the reference's TimestepNormState bit for bit
(proj/src/selection.cpp:13-31), so selections are identical and outputs agree
to the attention tolerance: float64 1e-9, float32 1e-5 relative."""
import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("norm_mode,slope_order", [("timestep_norm", "norm_then_slope"),
                                                   ("timestep_norm", "slope_then_norm"),
                                                   ("none", "norm_then_slope")])
def test_score_continue_equals_one_shot(cuda, norm_mode, slope_order):
    import torch

    from paper_2406_16747_b200 import ops

    B, L, D = 3, 257, 48
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.normal(size=(B, L, D))).to(cuda)
    w = torch.from_numpy(rng.normal(size=D)).to(cuda)
    sc = ops.ScoringConfig(norm_mode=norm_mode, slope_order=slope_order)
    raw, u, _, _ = ops.score_fwd(x, w, sc)
    st = torch.zeros((B, 3), dtype=torch.float64, device=cuda)
    parts, i = [], 0
    for n in (1, 100, 1, 55, 100):
        parts.append(ops.score_continue(x[:, i:i + n], w, sc, st))
        i += n
    assert torch.equal(torch.cat([p[1] for p in parts], 1), u)
    assert torch.equal(torch.cat([p[0] for p in parts], 1), raw)
    assert st[:, 0].tolist() == [float(L)] * B


CASES = [
    # L, D, heads, k, w, key, mask, prompt
    (96, 32, 2, 10.5, 8, "hard", "soft", 40),
    (80, 64, 4, 6.0, 0, "soft", "soft", 0),
    (120, 32, 1, 20.0, 16, "hard", "straight_through", 1),
    (70, 32, 2, 0.0, 12, "hard", "soft", 30),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_session_matches_reference_generate_step(cuda, reference, case, dtype):
    import torch

    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200 import DecodeSession, ops

    L, D, H, k, w, km, mm, prompt = case
    rng = np.random.default_rng(L + D)
    x = rng.normal(size=(L, D))
    ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
    wsc = rng.normal(size=D)
    f32 = dtype == "f32"
    if f32:  # the reference's float build sees the float-rounded inputs
        x = x.astype(np.float32).astype(np.float64)
        ws = [a.astype(np.float32).astype(np.float64) for a in ws]
    y_ref, peak = reference.decode(x, *ws, wsc, ref_cfg(k, w, heads=H, key_mode=km, mask_mode=mm),
                                   prompt, use_float=f32)
    tdt = torch.float32 if f32 else torch.float64
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda).to(tdt)
    cfg = ops.AttnConfig(k=k, window=w, key_mode=km, mask_mode=mm)
    s = DecodeSession(*(t(a) for a in ws), torch.from_numpy(wsc).to(cuda), cfg, H, batch=1,
                      max_len=L)
    xt = t(x)
    ys = []
    if prompt:
        ys.append(s.prefill(xt[None, :prompt])[0])
    for i in range(prompt, L):
        ys.append(s.step(xt[i][None])[0][None])
    y = torch.cat(ys, 0).double().cpu().numpy()
    tol = 1e-5 if f32 else 1e-9
    assert rel_err(y, y_ref) < tol, rel_err(y, y_ref)
    assert s.cache.state(0)["peak"] == peak or k == 0.0


def test_session_batch_of_sequences(cuda, reference):
    """B sequences in one session = B independent reference caches."""
    import torch

    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200 import DecodeSession, ops

    B, L, D, H, k, w, prompt = 3, 64, 32, 2, 8.5, 6, 17
    rng = np.random.default_rng(77)
    x = rng.normal(size=(B, L, D))
    ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
    wsc = rng.normal(size=D)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    s = DecodeSession(*(t(a) for a in ws), t(wsc), ops.AttnConfig(k=k, window=w), H, batch=B,
                      max_len=L)
    xt = t(x)
    ys = [s.prefill(xt[:, :prompt])] + [s.step(xt[:, i])[:, None] for i in range(prompt, L)]
    y = torch.cat(ys, 1).cpu().numpy()
    for b in range(B):
        y_ref, _ = reference.decode(x[b], *ws, wsc, ref_cfg(k, w, heads=H), prompt)
        assert rel_err(y[b], y_ref) < 1e-9, (b, rel_err(y[b], y_ref))


def test_session_forward_chunk_continues_state(cuda, reference):
    """forward_chunk onto a non-empty cache (Algorithm 3's recurrence): prompt,
    then a multi-row chunk, then single steps = the reference's forward_chunk
    followed by generate_step (the group size is invisible in the output,
    proj/src/cache.cpp:315-317)."""
    import torch

    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200 import DecodeSession, ops

    B, L, D, H, k, w, prompt, mid = 2, 80, 32, 2, 8.5, 6, 17, 40
    rng = np.random.default_rng(78)
    x = rng.normal(size=(B, L, D))
    ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
    wsc = rng.normal(size=D)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    s = DecodeSession(*(t(a) for a in ws), t(wsc), ops.AttnConfig(k=k, window=w), H, batch=B,
                      max_len=L)
    xt = t(x)
    ys = [s.forward_chunk(xt[:, :prompt]), s.forward_chunk(xt[:, prompt:mid])]
    ys += [s.step(xt[:, i])[:, None] for i in range(mid, L)]
    y = torch.cat(ys, 1).cpu().numpy()
    for b in range(B):
        y_ref, _ = reference.decode(x[b], *ws, wsc, ref_cfg(k, w, heads=H), prompt)
        assert rel_err(y[b], y_ref) < 1e-9, (b, rel_err(y[b], y_ref))
