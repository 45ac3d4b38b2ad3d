"""The fused projection GEMM + score (§8f row 2, skb_proj.cu): q|k|v = x W*
(hand-written tcgen05 GEMM; proj/src/cache.cpp:204-206) against an fp32
matmul of the same bf16 operands, and the score formed from the same x tiles
bit-identical to K1 (skb_score_fwd, itself bit-identical to the reference's
score_one, proj/include/sparsek/selection.hpp:69-96) — including row counts
that are not a multiple of the 128-row tile and the streaming Welford."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,L,D", [(1, 256, 256), (2, 1000, 512), (3, 77, 1024), (1, 4096, 768)])
@pytest.mark.parametrize("with_score", [True, False])
def test_proj_score_vs_reference_math(cuda, B, L, D, with_score):
    import torch

    from paper_2406_16747_b200 import ops

    g = torch.Generator(device=cuda)
    g.manual_seed(B * L + D)
    x = torch.randn((B, L, D), generator=g, device=cuda).to(torch.bfloat16)
    ws = [(torch.randn((D, D), generator=g, device=cuda) / D ** 0.5).to(torch.bfloat16) for _ in range(3)]
    wsc = torch.randn((D,), generator=g, device=cuda, dtype=torch.float64) / D ** 0.5
    sc = ops.ScoringConfig()
    q, k, v, raw, u, mean, sdev = ops.proj_score(x, *ws, wsc if with_score else None, sc)
    for out, w in zip((q, k, v), ws):
        ref = x.float() @ w.float()
        err = (out.float() - ref).norm() / ref.norm()
        assert err < 5e-3, float(err)
    if with_score:
        r_raw, r_u, r_mean, r_sdev = ops.score_fwd(x, wsc, sc)
        for a_, b_ in ((raw, r_raw), (u, r_u), (mean, r_mean), (sdev, r_sdev)):
            np.testing.assert_array_equal(a_.cpu().numpy(), b_.cpu().numpy())
    else:
        assert raw is None


def test_proj_score_nonfinite_raises(cuda):
    import torch

    from paper_2406_16747_b200 import NumericError, ops

    B, L, D = 1, 300, 256
    x = torch.randn((B, L, D), device=cuda).to(torch.bfloat16)
    x[0, 123, 7] = float("inf")
    ws = [torch.randn((D, D), device=cuda).to(torch.bfloat16) for _ in range(3)]
    with pytest.raises(NumericError):
        ops.proj_score(x, *ws, torch.ones(D, device=cuda, dtype=torch.float64), ops.ScoringConfig())


def test_x_level_bf16_fused_front_matches_library_front(cuda):
    """attention_torch through the fused front (bf16, D % 256 == 0) = the same
    op composed from cuBLAS projections + K1 (forward and gradients)."""
    import torch

    from paper_2406_16747_b200 import api, ops

    B, L, D, H = 2, 640, 256, 2
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    x = torch.randn((B, L, D), generator=g, device=cuda).to(torch.bfloat16)
    ws = [(0.5 * torch.randn((D, D), generator=g, device=cuda) / D ** 0.5).to(torch.bfloat16) for _ in range(4)]
    wsc = (torch.randn((D,), generator=g, device=cuda, dtype=torch.float64) / D ** 0.5)
    go = torch.randn((B, L, D), generator=g, device=cuda).to(torch.bfloat16)
    cfg = ops.AttnConfig(k=40.0, window=32)
    sc = ops.ScoringConfig()

    def run(fused):
        leaves = [t.clone().requires_grad_(True) for t in [x] + ws + [wsc]]
        xt, wq, wk, wv, wo, ws_ = leaves
        if fused:
            api._FUSED_FRONT = True
            try:
                y, _ = api.attention_torch(xt, wq, wk, wv, wo, ws_, cfg, H, sc)
            finally:
                api._FUSED_FRONT = False
        else:
            p = D // H
            q, k, v = ((xt @ w).view(B, L, H, p) for w in (wq, wk, wv))
            u = ops.score_tokens(xt, ws_, sc)
            hc = ops.sparsek_attention_core(q, k, v, u, cfg)
            y = hc.reshape(B, L, D) @ wo
        y.backward(go)
        return [y.detach()] + [t.grad for t in leaves]

    a, b = run(True), run(False)
    names = ["y", "dx", "dwq", "dwk", "dwv", "dwo", "dw_score"]
    for n, ta, tb in zip(names, a, b):
        err = (ta.double() - tb.double()).norm() / tb.double().norm()
        assert err < 2e-2, (n, float(err))
