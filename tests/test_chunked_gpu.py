"""GPU: chunk-wise recurrent training (Algorithm 3).

The reference's chunked_forward (proj/src/cache.cpp:548-563) reproduces the
unchunked forward exactly (proj/tests/test_cache.cpp:34-64) and its backward
never lets a gradient cross to the left of a chunk start
(proj/src/attention.cpp:228-234, 284-300, 472, 491). Checked against the
compiled reference at the x level in float64, and the bf16 tensor-core
backward against the f32 gather path with chunking on."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2406_16747_b200 as sparsek  # noqa: E402


@pytest.mark.parametrize("chunk", [40, 64, 97])
@pytest.mark.parametrize("km,mm", [("hard", "soft"), ("soft", "straight_through")])
def test_chunked_x_level_vs_reference(cuda, reference, chunk, km, mm):
    from oracle.oracle import ref_cfg

    rng = np.random.default_rng(chunk)
    L, D, H = 200, 32, 4
    x = rng.normal(size=(L, D))
    s = 0.6 / np.sqrt(D)
    wq, wk, wv, wo = (s * rng.normal(size=(D, D)) for _ in range(4))
    ws = rng.normal(size=D) / np.sqrt(D)
    go = rng.normal(size=(L, D))
    k, w = 12.5, 10
    tape, grads = reference.attention(x, wq, wk, wv, wo, ws, ref_cfg(k, w, heads=H, key_mode=km,
                                                                    mask_mode=mm),
                                      grad_out=go, chunk_len=chunk)
    y, g = sparsek.attention_grads(x, wq, wk, wv, wo, ws, k, w, go, heads=H, key_mode=km,
                                   mask_mode=mm, chunk_len=chunk)
    np.testing.assert_allclose(y, tape.y, rtol=1e-9, atol=1e-11)
    y2 = sparsek.chunked_forward(x, chunk, wq, wk, wv, wo, ws, k, w, heads=H, key_mode=km,
                                 mask_mode=mm)
    np.testing.assert_allclose(y2, tape.y, rtol=1e-9, atol=1e-11)
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dw_score"):
        a, b = g[name], grads[name]
        assert np.linalg.norm(a - b) <= 1e-8 * max(np.linalg.norm(b), 1e-12), name
    # the stop-gradient is real: the unchunked gradients differ
    _, g0 = sparsek.attention_grads(x, wq, wk, wv, wo, ws, k, w, go, heads=H, key_mode=km,
                                    mask_mode=mm)
    assert np.linalg.norm(g0["dwk"] - g["dwk"]) > 1e-6 * np.linalg.norm(g0["dwk"])


@pytest.mark.parametrize("chunk", [256, 1000])
def test_chunked_tensor_core_vs_gather(cuda, chunk):
    import torch

    from paper_2406_16747_b200 import ops

    B, L, H, p, k, w = 1, 2048, 2, 128, 300.0, 300
    g = torch.Generator(device=cuda)
    g.manual_seed(chunk)
    q, kk, v, do = (torch.randn((B, L, H, p), generator=g, device=cuda).to(torch.bfloat16)
                    for _ in range(4))
    u = (torch.randn((B, L), generator=g, device=cuda, dtype=torch.float64)
         + 0.01 * torch.arange(1, L + 1, device=cuda, dtype=torch.float64))
    res = {}
    for fg in (False, True):
        cfg = ops.AttnConfig(k=k, window=w, chunk_len=chunk, force_gather=fg)
        cast = (lambda t: t.float().contiguous()) if fg else (lambda t: t)
        o, lse, sel = ops.attn_fwd(cast(q), cast(kk), cast(v), u, cfg)
        res[fg] = (o,) + tuple(ops.attn_bwd(cast(q), cast(kk), cast(v), o, cast(do), lse, u, sel, cfg))
    torch.cuda.synchronize()
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))
    for nm, a, b in zip(("o", "dq", "dk", "dv", "du"), res[False], res[True]):
        assert rel(a, b) < 2e-2, (nm, rel(a, b))
