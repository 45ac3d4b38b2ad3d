"""K1 scoring (proj/include/sparsek/selection.hpp:69-96, Welford
proj/src/selection.cpp:13-20) at model width: raw = x.w and the normalised
scores u must be bit-identical to the C oracle (itself pinned bit-exact to
the reference, tests/test_oracle.py) for every x dtype, for 16-byte aligned
rows (the staged HBM-streaming kernel) and unaligned rows (the row-per-thread
fallback), and over long sequences (the Welford division runs as a
reciprocal + fma correction that must equal the correctly rounded quotient)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
@pytest.mark.parametrize("L,D", [(3000, 4096), (257, 768), (130, 1001)])
def test_score_bit_identical_at_width(cuda, oracle, dtype, L, D):
    import torch

    from paper_2406_16747_b200 import ops

    rng = np.random.default_rng(L + D)
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dtype]
    B = 2
    x = torch.from_numpy(rng.normal(size=(B, L, D))).to(tdt)
    w = rng.normal(size=D) / np.sqrt(D)
    sc = ops.ScoringConfig()
    raw, u, mean, sdev = ops.score_fwd(x.to(cuda), torch.from_numpy(w).to(cuda), sc)
    xn = x.double().numpy()
    for b in range(B):
        r_raw, r_u, r_mean, r_sdev = oracle.score_fwd(xn[b], w)
        np.testing.assert_array_equal(raw[b].cpu().numpy(), r_raw)
        np.testing.assert_array_equal(u[b].cpu().numpy(), r_u)
        np.testing.assert_array_equal(mean[b].cpu().numpy(), r_mean)
        np.testing.assert_array_equal(sdev[b].cpu().numpy(), r_sdev)


@pytest.mark.parametrize("slope_order", [0, 1])
def test_welford_long_sequence_bit_identical(cuda, oracle, slope_order):
    import torch

    from paper_2406_16747_b200 import ops

    L = 200_000
    rng = np.random.default_rng(slope_order)
    # heavy-tailed raw values (wide exponent range) plus exact repeats and zeros
    xr = rng.standard_cauchy(size=L) * 10.0 ** rng.integers(-6, 6, size=L)
    xr[::97] = 0.0
    xr[1::89] = xr[::89][: len(xr[1::89])]
    x = torch.from_numpy(xr.reshape(1, L, 1))
    w = np.array([1.0])
    sc = ops.ScoringConfig(slope_order="slope_then_norm" if slope_order == 0 else "norm_then_slope")
    raw, u, mean, sdev = ops.score_fwd(x.to(cuda), torch.from_numpy(w).to(cuda), sc)
    r_raw, r_u, r_mean, r_sdev = oracle.score_fwd(xr.reshape(L, 1), w, slope_order=slope_order)
    np.testing.assert_array_equal(mean[0].cpu().numpy(), r_mean)
    np.testing.assert_array_equal(sdev[0].cpu().numpy(), r_sdev)
    np.testing.assert_array_equal(u[0].cpu().numpy(), r_u)
