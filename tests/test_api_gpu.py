"""GPU: the reference's Python smoke suite (proj/tests/python/test_smoke.py),
run against paper_2406_16747_b200 as a drop-in for `import sparsek`, plus the
x-level forward/backward against the compiled reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2406_16747_b200 as sparsek  # noqa: E402


def test_documented_example(cuda):
    sol = sparsek.sparsek([0.9, 0.5, 0.1], 2.0)
    np.testing.assert_allclose(sol["p"], [1.0, 0.7, 0.3], atol=1e-12)
    assert sol["tau"] == pytest.approx(-0.2)
    assert sol["u_count"] == 1


def test_budget_saturates_everything(cuda):
    sol = sparsek.sparsek([3.0, -1.0], 5.0)
    np.testing.assert_allclose(sol["p"], [1.0, 1.0])
    assert sol["tau"] is None


def test_jvp_matches_support_mean_formula(cuda):
    z = [0.9, 0.5, 0.1]
    v = [0.3, -0.2, 0.5]
    jvp = sparsek.sparsek_jvp(z, 2.0, v)
    mean = (v[1] + v[2]) / 2.0
    np.testing.assert_allclose(jvp, [0.0, v[1] - mean, v[2] - mean], atol=1e-12)


def test_stream_prefix_equals_batch(cuda):
    rng = np.random.default_rng(5)
    z = rng.normal(size=40)
    st = sparsek.Stream(4.0)
    for t in range(len(z)):
        st.push(z[t])
        inc = st.solution()
        batch = sparsek.sparsek(list(z[: t + 1]), 4.0)
        np.testing.assert_allclose(inc["p"], batch["p"], atol=1e-9)
    assert st.t == len(z)


def test_errors_are_python_exceptions(cuda):
    with pytest.raises(ValueError):
        sparsek.sparsek([1.0, 2.0], -1.0)
    with pytest.raises(ValueError):
        sparsek.sparsek_jvp([1.0, 2.0], 1.0, [0.5])
    with pytest.raises(ArithmeticError):
        sparsek.sparsek([1.0, float("nan")], 1.0)


def test_attention_matches_dense_when_budget_covers_all(cuda):
    rng = np.random.default_rng(11)
    n, d, heads = 12, 8, 2
    x = rng.normal(size=(n, d))
    wq, wk, wv, wo = (0.2 * rng.normal(size=(d, d)) for _ in range(4))
    w_score = list(0.2 * rng.normal(size=d))
    out = sparsek.attention(x, wq, wk, wv, wo, w_score, k=float(n), window=2, heads=heads)
    dense = sparsek.dense_attention(x, wq, wk, wv, wo, heads=heads)
    np.testing.assert_allclose(out, dense, atol=1e-9)
    assert out.shape == (n, d)


@pytest.mark.parametrize("z_kind", ["normal", "ties", "constant", "ramp"])
@pytest.mark.parametrize("k", [1.0, 2.5, 7.0, 60.0])
def test_operator_vs_reference(cuda, reference, z_kind, k):
    rng = np.random.default_rng(3)
    m = 300
    z = {"normal": rng.normal(size=m), "ties": 0.25 * rng.integers(-8, 9, size=m),
         "constant": np.full(m, 0.9), "ramp": 0.05 * np.arange(m)}[z_kind]
    a, b = sparsek.sparsek(z, k), reference.sparsek(z, k)
    np.testing.assert_allclose(a["p"], b["p"], atol=1e-12)
    if b["infeasible"]:
        assert a["tau"] is None
    elif not b["degenerate"]:
        assert a["tau"] == pytest.approx(b["tau"], rel=1e-12, abs=1e-12)
    assert (a["u_count"], a["w_count"]) == (b["u_count"], b["w_count"])
    v = rng.normal(size=m)
    np.testing.assert_allclose(sparsek.sparsek_jvp(z, k, v), reference.sparsek_jvp(z, k, v),
                               atol=1e-12)
    np.testing.assert_array_equal(sparsek.topk_hard(z, int(k)), reference.topk_hard(z, int(k)))


@pytest.mark.parametrize("km,mm", [("hard", "soft"), ("soft", "straight_through")])
def test_x_level_forward_backward_vs_reference(cuda, reference, km, mm):
    """sparsek_attention + sparsek_attention_backward through x and the D x D
    projections, float64, against the reference library."""
    from oracle.oracle import ref_cfg

    rng = np.random.default_rng(21)
    L, D, H = 200, 32, 4
    x = rng.normal(size=(L, D))
    s = 0.6 / np.sqrt(D)
    wq, wk, wv, wo = (s * rng.normal(size=(D, D)) for _ in range(4))
    ws = rng.normal(size=D) / np.sqrt(D)
    go = rng.normal(size=(L, D))
    k, w = 12.5, 10
    tape, grads = reference.attention(x, wq, wk, wv, wo, ws, ref_cfg(k, w, heads=H, key_mode=km,
                                                                    mask_mode=mm), grad_out=go)
    y, g = sparsek.attention_grads(x, wq, wk, wv, wo, ws, k, w, go, heads=H, key_mode=km,
                                   mask_mode=mm)
    np.testing.assert_allclose(y, tape.y, rtol=1e-9, atol=1e-11)
    y2 = sparsek.attention(x, wq, wk, wv, wo, ws, k, w, heads=H, key_mode=km, mask_mode=mm)
    np.testing.assert_allclose(y2, tape.y, rtol=1e-9, atol=1e-11)
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dw_score"):
        a, b = g[name], grads[name]
        assert np.linalg.norm(a - b) <= 1e-8 * max(np.linalg.norm(b), 1e-12), name
