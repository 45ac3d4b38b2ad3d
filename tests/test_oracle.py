"""CPU: pin the oracle (oracle/sparsek_oracle.c) to the reference.

Three anchors: (1) the reference's own known-answer vectors
(proj/tests/test_sparsek_op.cpp:131-177,257-283, proj/tests/python/test_smoke.py),
(2) the compiled reference itself (oracle/_ref, when present), bit for bit,
(3) the committed golden fixtures generated from the reference
(tests/golden/make_golden.py), which travel to the GPU box.
"""
import math

import numpy as np
import pytest

from tests.helpers import golden_cases, load_golden


# ------------------------------------------------------------ known answers
def test_frozen_three_values_budget_two(oracle):
    s = oracle.sparsek([0.9, 0.5, 0.1], 2.0)
    np.testing.assert_allclose(s["p"], [1.0, 0.7, 0.3], atol=1e-12)
    assert s["tau"] == pytest.approx(-0.2, abs=1e-12)
    assert (s["u_count"], s["w_count"]) == (1, 3)
    assert not s["degenerate"] and not s["infeasible"]


def test_frozen_constant_values(oracle):
    s = oracle.sparsek([0.4, 0.4, 0.4], 2.0)
    np.testing.assert_allclose(s["p"], [2 / 3] * 3, atol=1e-12)
    assert s["tau"] == pytest.approx(0.4 - 2 / 3, abs=1e-12)


def test_frozen_dominant_value_degenerate(oracle):
    s = oracle.sparsek([2.0, 0.0, 0.0], 1.0)
    np.testing.assert_array_equal(s["p"], [1.0, 0.0, 0.0])
    assert s["degenerate"] and 0.0 <= s["tau"] <= 1.0


def test_infeasible_saturates(oracle):
    s = oracle.sparsek([0.3, -0.1], 5.0)
    assert s["infeasible"] and s["tau"] == -math.inf
    np.testing.assert_array_equal(s["p"], [1.0, 1.0])


def test_jvp_known(oracle):
    np.testing.assert_allclose(oracle.sparsek_jvp([0.9, 0.5, 0.1], 2.0, [0.0, 4.0, 2.0]),
                               [0.0, 1.0, -1.0], atol=1e-12)


def test_topk_ties_lower_index(oracle):
    np.testing.assert_array_equal(oracle.topk_hard([0.5, 0.9, 0.5, 0.1], 2), [1, 1, 0, 0])


def test_stream_rejects_below_tau(oracle):
    z = [5.0, 4.0, 3.0, 2.0]
    tau, ins = oracle.stream_taus(z, 2.0)
    t = tau[-1]
    tau2, ins2 = oracle.stream_taus(z + [t - 1.0, t + 0.5], 2.0)
    assert not ins2[4] and tau2[4] == t and ins2[5]


# ------------------------------------------------------ against the reference
def _flavor(rng, m, f):
    if f == 0:
        return rng.normal(size=m)
    if f == 1:
        return rng.uniform(-3, 3, size=m)
    if f == 2:
        return 0.25 * rng.integers(-8, 9, size=m)
    if f == 3:
        return np.full(m, 0.9)
    return 0.05 * np.arange(m) + 0.01 * rng.normal(size=m)


@pytest.mark.parametrize("flavor", range(5))
def test_sparsek_matches_reference(oracle, reference, flavor):
    rng = np.random.default_rng(100 + flavor)
    for m in (1, 2, 7, 33, 200):
        for k in (0.5, 1.0, 2.5, 4.0, 17.0):
            z = _flavor(rng, m, flavor)
            a, b = oracle.sparsek(z, k), reference.sparsek(z, k)
            np.testing.assert_array_equal(a["p"], b["p"])
            assert a["tau"] == b["tau"]
            assert (a["u_count"], a["w_count"]) == (b["u_count"], b["w_count"])
            v = rng.normal(size=m)
            np.testing.assert_array_equal(oracle.sparsek_jvp(z, k, v), reference.sparsek_jvp(z, k, v))
            kk = int(rng.integers(0, m + 2))
            np.testing.assert_array_equal(oracle.topk_hard(z, kk), reference.topk_hard(z, kk))


@pytest.mark.parametrize("flavor", range(5))
def test_stream_taus_bit_exact(oracle, reference, flavor):
    rng = np.random.default_rng(7 + flavor)
    z = _flavor(rng, 600, flavor)
    for k in (1.0, 3.0, 4.5, 40.0):
        a, ia = oracle.stream_taus(z, k)
        b, ib, _, _ = reference.stream(z, k)
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(ia, ib)


CORE_CASES = [
    # H, p, k, w, key, mask, norm, slope
    (2, 32, 8.5, 8, "hard", "soft", "none", False),
    (2, 32, 8.0, 8, "soft", "soft", "timestep_norm", True),
    (2, 32, 6.0, 0, "hard", "straight_through", "none", True),
    (4, 16, 3.5, 5, "soft", "straight_through", "timestep_norm", True),
    (2, 64, 16.0, 16, "hard", "soft", "timestep_norm", True),
]


@pytest.mark.parametrize("case", CORE_CASES)
def test_core_matches_reference_bit_exact(oracle, reference, case):
    from oracle.oracle import core_problem_via_reference

    H, p, k, w, km, mm, nm, slope = case
    L = H * p
    rng = np.random.default_rng(hash(case) % 2**32)
    Q, K, V, dO = (rng.normal(size=(L, H, p)) for _ in range(4))
    ws = rng.normal(size=L)
    tape, grads = core_problem_via_reference(reference, Q, K, V, ws, dO, kbudget=k, window=w,
                                             key_mode=km, mask_mode=mm, norm_mode=nm,
                                             slope_enabled=slope)
    norm = int(nm == "timestep_norm")
    raw, u, mean, sdev = oracle.score_fwd(np.eye(L), ws, norm_mode=norm, slope_enabled=slope)
    np.testing.assert_array_equal(u, tape.u)
    sel = oracle.select(u, k, w)
    np.testing.assert_array_equal(sel.att_off, tape.att_off)
    np.testing.assert_array_equal(sel.att, tape.att)
    np.testing.assert_array_equal(sel.n_sel, tape.n_sel)
    np.testing.assert_array_equal(sel.tau_q[w:], tape.tau_push[: L - w])
    o, maxa, den = oracle.attn_fwd(Q, K, V, sel, kbudget=k, window=w, key_mode=km, mask_mode=mm)
    np.testing.assert_array_equal(o.reshape(L, -1), tape.head_concat)
    np.testing.assert_array_equal(maxa, tape.maxa)
    np.testing.assert_array_equal(den, tape.denom)
    dq, dk, dv, gu = oracle.attn_bwd(Q, K, V, dO, u, sel, maxa, den, kbudget=k, window=w,
                                     key_mode=km, mask_mode=mm)
    np.testing.assert_array_equal(dq.reshape(L, -1), grads["dwq"])
    np.testing.assert_array_equal(dk.reshape(L, -1), grads["dwk"])
    np.testing.assert_array_equal(dv.reshape(L, -1), grads["dwv"])
    graw = oracle.score_bwd(gu, raw, mean, sdev, norm_mode=norm)
    np.testing.assert_array_equal(graw, grads["dw_score"])


def test_selection_is_brute_force_top_floor_k(oracle):
    """Retention == top-floor(k) of the exited prefix, ties to the lower index
    (proj/tests/test_cache.cpp:84-97)."""
    rng = np.random.default_rng(67)
    for u in (rng.normal(size=300), 0.5 * rng.integers(-3, 4, size=300).astype(float)):
        for k, w in ((8.5, 8), (24.0, 16), (5.0, 0)):
            sel = oracle.select(u, k, w)
            kf = int(math.floor(k))
            for i in range(len(u)):
                t = i - w
                if t < 0:
                    assert sel.n_sel[i] == 0
                    continue
                order = sorted(range(t + 1), key=lambda j: (-u[j], j))[:kf]
                np.testing.assert_array_equal(sel.sel_of(i), sorted(order))


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_oracle_reproduces_golden(oracle, path):
    g = load_golden(path)
    H, p, k, w = g["H"], g["p"], g["k"], g["w"]
    L = H * p
    norm = int(g["norm_mode"] == "timestep_norm")
    raw, u, mean, sdev = oracle.score_fwd(np.eye(L), g["w_score"], norm_mode=norm,
                                          slope_enabled=bool(g["slope"]))
    np.testing.assert_array_equal(u, g["u"])
    sel = oracle.select(u, k, w)
    np.testing.assert_array_equal(sel.att, g["att"])
    o, maxa, den = oracle.attn_fwd(g["Q"], g["K"], g["V"], sel, kbudget=k, window=w,
                                   key_mode=g["key_mode"], mask_mode=g["mask_mode"])
    np.testing.assert_array_equal(o.reshape(L, -1), g["head_concat"])
    dq, dk, dv, gu = oracle.attn_bwd(g["Q"], g["K"], g["V"], g["dO"], u, sel, maxa, den,
                                     kbudget=k, window=w, key_mode=g["key_mode"],
                                     mask_mode=g["mask_mode"])
    np.testing.assert_array_equal(dq.reshape(L, -1), g["dq"])
    graw = oracle.score_bwd(gu, raw, mean, sdev, norm_mode=norm)
    np.testing.assert_array_equal(graw, g["dw_score"])
