"""Linear-attention mix (Appendix B.1, §8f row 4) against the compiled
reference: linear_mix_attention forward and sparsek_attention_backward with
LinearMixParams (proj/src/cache.cpp:262-278,322-356; proj/src/attention.cpp:
317-445,519-549), every gradient including dfeat, in the reference's double
and float instantiations; the softmax limit of proj/tests/test_attention.cpp:
296-330 (every gate 1: the mixture is plain causal softmax attention)."""
import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

CASES = [
    # L, D, H, k, window, chunk
    (48, 16, 2, 6.5, 4, 0),
    (64, 24, 3, 9.0, 0, 0),      # no window: the linear branch covers the query itself
    (40, 16, 2, 0.0, 5, 0),      # scores idle: window + linear
    (56, 16, 1, 0.0, 0, 0),      # pure linear attention
    (72, 16, 2, 7.25, 6, 24),    # chunk-wise (Algorithm 3): key-side gradients stay in the chunk
    (90, 32, 2, 20.0, 8, 0),
]


def _problem(L, D, H, seed):
    rng = np.random.default_rng(seed)
    p = D // H
    x = rng.normal(size=(L, D))
    s = 0.5 / np.sqrt(D)
    ws = [s * rng.normal(size=(D, D)) for _ in range(4)]
    wsc = rng.normal(size=D) / np.sqrt(D)
    feat = rng.normal(size=(H, p, p)) / np.sqrt(p)
    go = rng.normal(size=(L, D))
    return x, ws, wsc, feat, go


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_linear_mix_f64_vs_reference(cuda, reference, case):
    import paper_2406_16747_b200 as sk
    from oracle.oracle import ref_cfg

    L, D, H, k, w, chunk = case
    x, ws, wsc, feat, go = _problem(L, D, H, L + D)
    y_ref, g_ref = reference.linear_mix(x, *ws, wsc, feat, ref_cfg(k, w, heads=H), grad_out=go,
                                        chunk_len=chunk)
    if chunk == 0:
        y = sk.linear_mix_attention(x, *ws, wsc, feat, k, w, heads=H)
        assert rel_err(y, y_ref) < 1e-10, rel_err(y, y_ref)
    y2, g = sk.linear_mix_attention_grads(x, *ws, wsc, feat, k, w, go, heads=H, chunk_len=chunk)
    assert rel_err(y2, y_ref) < 1e-10
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dw_score", "dfeat"):
        if name == "dw_score" and k == 0.0:
            continue
        assert rel_err(g[name], g_ref[name]) < 1e-9, (name, rel_err(g[name], g_ref[name]))


@pytest.mark.parametrize("case", CASES[:3], ids=[str(c) for c in CASES[:3]])
def test_linear_mix_core_f32_vs_reference_float(cuda, reference, case):
    """The float instantiation: core q/k/v/u in float32 (the reference's float
    path rounds q/k/v to float; its scores and gates stay double)."""
    import torch

    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200 import ops

    L, D, H, k, w, chunk = case
    x, ws, wsc, feat, go = _problem(L, D, H, 7 * L)
    p = D // H
    x32 = x.astype(np.float32).astype(np.float64)
    ws32 = [a.astype(np.float32).astype(np.float64) for a in ws]
    f32 = feat.astype(np.float32).astype(np.float64)
    y_ref, _ = reference.linear_mix(x32, *ws32, wsc, f32, ref_cfg(k, w, heads=H), use_float=True)
    dev = cuda
    t = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dt)
    xt = t(x32).view(1, L, D)
    q, kk, v = ((xt @ t(wm)).view(1, L, H, p).contiguous() for wm in ws32[:3])
    sc = ops.ScoringConfig()
    u = ops.score_fwd(t(x32, torch.float64).view(1, L, D), t(wsc, torch.float64), sc)[1] if k > 0 else \
        torch.zeros((1, L), dtype=torch.float64, device=dev)
    cfg = ops.AttnConfig(k=k, window=w, linear_mix=True)
    o, den, _ = ops.linmix_fwd(q, kk, v, u, t(f32, torch.float64), cfg)
    y = (o.reshape(L, D) @ t(ws32[3])).double().cpu().numpy()
    assert rel_err(y, y_ref) < 1e-5, rel_err(y, y_ref)


def test_linear_mix_softmax_limit(cuda):
    """Budget covering every position (all gates 1): the mixture is causal
    softmax attention (proj/tests/test_attention.cpp:296-330)."""
    import paper_2406_16747_b200 as sk

    L, D, H = 50, 16, 2
    x, ws, wsc, feat, _ = _problem(L, D, H, 3)
    y = sk.linear_mix_attention(x, *ws, wsc, feat, float(L + 5), 1, heads=H)
    dense = sk.dense_attention(x, *ws, heads=H)
    np.testing.assert_allclose(y, dense, rtol=0, atol=1e-10)


def test_linear_mix_errors(cuda):
    import paper_2406_16747_b200 as sk

    L, D, H = 20, 8, 2
    x, ws, wsc, feat, _ = _problem(L, D, H, 4)
    with pytest.raises(ValueError):  # one feature map per head
        sk.linear_mix_attention(x, *ws, wsc, feat[:1], 4.0, 2, heads=H)
    with pytest.raises(ValueError):  # head_dim x head_dim
        sk.linear_mix_attention(x, *ws, wsc, feat[:, :2, :2], 4.0, 2, heads=H)
    with pytest.raises(ValueError):  # w_score length
        sk.linear_mix_attention(x, *ws, wsc[:3], feat, 4.0, 2, heads=H)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("k,w,prompt", [(6.5, 4, 20), (9.0, 0, 1), (0.0, 5, 12)])
def test_linear_mix_decode_vs_reference(cuda, reference, dtype, k, w, prompt):
    """Incremental decoding with the linear mix: the cache carries phi(k) of its
    rows and the prefix state M, b across steps (forward_chunk / generate_step
    with LinearMixParams, proj/src/cache.cpp:262-278,322-356,570-577)."""
    import torch

    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200 import DecodeSession, ops

    L, D, H = 56, 16, 2
    x, ws, wsc, feat, _ = _problem(L, D, H, 11 + prompt)
    tdt = {"f64": torch.float64, "f32": torch.float32}[dtype]
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
        ws = [a.astype(np.float32).astype(np.float64) for a in ws]
        feat = feat.astype(np.float32).astype(np.float64)
    y_ref = reference.linear_mix_decode(x, *ws, wsc, feat, ref_cfg(k, w, heads=H), prompt,
                                        use_float=dtype == "f32")
    t = lambda a, dt=tdt: torch.from_numpy(np.ascontiguousarray(a)).to(cuda).to(dt)
    s = DecodeSession(*(t(a) for a in ws), t(wsc) if k > 0 else None, ops.AttnConfig(k=k, window=w), H,
                      batch=1, max_len=L, dtype=tdt, feat=t(feat, torch.float64))
    xt = t(x).view(1, L, D)
    ys = [s.forward_chunk(xt[:, :prompt])] + [s.step(xt[:, i])[:, None] for i in range(prompt, L)]
    y = torch.cat(ys, 1)[0].double().cpu().numpy()
    tol = 1e-9 if dtype == "f64" else 1e-5
    assert rel_err(y, y_ref) < tol, rel_err(y, y_ref)
