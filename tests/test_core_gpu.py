"""GPU parity of the core path (K2 select, K3 fwd, K4 bwd + JVP, K1 score)
against the reference's golden fixtures and the C oracle.

Tolerances (north star): selected sets bit-exact; tau within 1e-9 relative on
non-degenerate steps (proj/tests/test_stream.cpp:50-51 compares tau the same
way); float64 outputs/gradients within 1e-9 relative, float32 within 1e-5,
bfloat16 within 2e-2.
"""
import math

import numpy as np
import pytest

from tests.helpers import golden_cases, load_golden, rel_err, run_core_gpu, sel_lists_from_leave

pytestmark = pytest.mark.gpu


def _check_selection(res, u, tau_ref_q, att_lists_ref, L, w, k):
    sel = sel_lists_from_leave(res["leave"], L, w)
    for i in range(L):
        np.testing.assert_array_equal(sel[i], att_lists_ref[i], err_msg=f"query {i}")
    # tau on non-degenerate steps; gates everywhere
    for i in range(w, L):
        tr, tg = tau_ref_q[i], res["tau_q"][i]
        if not math.isfinite(tr):
            assert not math.isfinite(tg), (i, tr, tg)
            continue
        t = i - w
        f = u[: t + 1] - tr
        if np.any((f > 0) & (f < 1)):
            assert abs(tg - tr) <= 1e-9 * max(1.0, abs(tr)), (i, tr, tg)
        ga = np.clip(u[sel[i]] - tg, 0, 1)
        gr = np.clip(u[sel[i]] - tr, 0, 1)
        np.testing.assert_allclose(ga, gr, rtol=0, atol=1e-9)


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_golden_f64(cuda, path):
    import torch

    from paper_2406_16747_b200 import ops

    g = load_golden(path)
    H, p, k, w = g["H"], g["p"], g["k"], g["w"]
    L = H * p
    # K1: scores bit-identical to the reference's
    x = torch.eye(L, dtype=torch.float64, device=cuda)[None]
    wsc = torch.from_numpy(g["w_score"]).to(cuda)
    sc = ops.ScoringConfig(slope_enabled=bool(g["slope"]), norm_mode=g["norm_mode"])
    raw, u, mean, sdev = ops.score_fwd(x, wsc, sc)
    np.testing.assert_array_equal(u[0].cpu().numpy(), g["u"])
    res = run_core_gpu(g["Q"], g["K"], g["V"], g["u"], g["dO"], k=k, w=w, key_mode=g["key_mode"],
                       mask_mode=g["mask_mode"], dtype="f64")
    att_ref = [g["att"][g["att_off"][i]: g["att_off"][i] + g["n_sel"][i]] for i in range(L)]
    tau_ref_q = np.full(L, -np.inf)
    tau_ref_q[w:] = g["tau_push"][: L - w]
    _check_selection(res, g["u"], tau_ref_q, att_ref, L, w, k)
    assert rel_err(res["o"].reshape(L, -1), g["head_concat"]) < 1e-10
    lse_ref = (g["maxa"] + np.log(g["denom"])).T  # [H, L]
    np.testing.assert_allclose(res["lse"], lse_ref, rtol=1e-11, atol=1e-11)
    assert rel_err(res["dq"].reshape(L, -1), g["dq"]) < 1e-9
    assert rel_err(res["dk"].reshape(L, -1), g["dk"]) < 1e-9
    assert rel_err(res["dv"].reshape(L, -1), g["dv"]) < 1e-9
    graw, dw = ops.score_bwd(x, wsc, sc, torch.from_numpy(res["du"][None]).to(cuda), raw, mean,
                             sdev)
    np.testing.assert_allclose(dw.cpu().numpy(), g["dw_score"], rtol=1e-8,
                               atol=1e-9 * np.abs(g["dw_score"]).max())


def _scores(rng, L, kind):
    if kind == "recency":
        return rng.normal(size=L) + 0.01 * np.arange(1, L + 1)
    if kind == "iid":
        return rng.normal(size=L)
    if kind == "ties":
        return 0.5 * rng.integers(-4, 5, size=L).astype(np.float64)
    if kind == "constant":
        return np.full(L, 0.25)
    if kind == "falling":
        return -0.01 * np.arange(L) + 0.3 * rng.normal(size=L)
    raise ValueError(kind)


def _oracle_core(oracle, Q, K, V, u, dO, k, w, km, mm):
    sel = oracle.select(u, k, w)
    o, maxa, den = oracle.attn_fwd(Q, K, V, sel, kbudget=k, window=w, key_mode=km, mask_mode=mm)
    dq, dk, dv, gu = oracle.attn_bwd(Q, K, V, dO, u, sel, maxa, den, kbudget=k, window=w,
                                     key_mode=km, mask_mode=mm)
    return sel, o, maxa + np.log(den), dq, dk, dv, gu


CASES = [
    # L, H, p, k, w, key, mask, kind
    (1024, 4, 64, 64.0, 64, "hard", "soft", "recency"),     # cfg1 shape
    (700, 2, 32, 24.5, 16, "soft", "soft", "iid"),
    (600, 2, 16, 17.0, 0, "hard", "straight_through", "ties"),
    (300, 1, 32, 9.0, 7, "soft", "straight_through", "constant"),
    (500, 3, 32, 40.0, 33, "hard", "soft", "falling"),
    (200, 2, 64, 300.0, 5, "hard", "soft", "iid"),          # budget covers everything
    (150, 2, 32, 0.0, 12, "hard", "soft", "iid"),           # pure window
    (90, 2, 32, 0.5, 6, "soft", "soft", "iid"),             # floor(k) = 0 with a stream
    (40, 1, 32, 8.0, 64, "hard", "soft", "iid"),            # L < w: no pushes
    (257, 2, 128, 32.0, 31, "hard", "soft", "recency"),
    # many tiles per query block: K/V/metadata rings wrap several times
    (2048, 2, 128, 300.0, 300, "hard", "soft", "recency"),
    (1536, 1, 64, 420.5, 200, "soft", "soft", "iid"),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_core_vs_oracle(cuda, oracle, case, dtype):
    L, H, p, k, w, km, mm, kind = case
    rng = np.random.default_rng(L * 7 + H)
    Q, K, V, dO = (rng.normal(size=(L, H, p)) for _ in range(4))
    u = _scores(rng, L, kind)
    if dtype == "bf16":  # compare against the oracle on the rounded inputs
        import torch

        rnd = lambda a: torch.from_numpy(a).to(torch.bfloat16).double().numpy()
        Q, K, V, dO = rnd(Q), rnd(K), rnd(V), rnd(dO)
    sel, o, lse, dq, dk, dv, gu = _oracle_core(oracle, Q, K, V, u, dO, k, w, km, mm)
    res = run_core_gpu(Q, K, V, u, dO, k=k, w=w, key_mode=km, mask_mode=mm, dtype=dtype)
    att_ref = [sel.sel_of(i) for i in range(L)]
    _check_selection(res, u, sel.tau_q, att_ref, L, w, k)
    tol = {"f64": 1e-10, "f32": 1e-5, "bf16": 2e-2}[dtype]
    assert rel_err(res["o"], o) < tol
    np.testing.assert_allclose(res["lse"], lse.T, rtol=0, atol=max(tol, 1e-9) * 10)
    gtol = {"f64": 1e-9, "f32": 1e-5, "bf16": 2e-2}[dtype]
    for name, a, b in (("dq", res["dq"], dq), ("dk", res["dk"], dk), ("dv", res["dv"], dv)):
        assert rel_err(a, b) < gtol, (name, rel_err(a, b))
    if np.abs(gu).max() > 0:
        assert rel_err(res["du"], gu) < (1e-8 if dtype == "f64" else gtol), rel_err(res["du"], gu)
    else:
        assert np.abs(res["du"]).max() == 0


def test_batched_sequences_are_independent(cuda, oracle):
    L, H, p, k, w = 400, 2, 32, 20.0, 10
    rng = np.random.default_rng(5)
    Q, K, V, dO = (rng.normal(size=(3, L, H, p)) for _ in range(4))
    u = np.stack([_scores(rng, L, kd) for kd in ("recency", "iid", "ties")])
    res = run_core_gpu(Q, K, V, u, dO, k=k, w=w, dtype="f64")
    for b in range(3):
        sel, o, lse, dq, dk, dv, gu = _oracle_core(oracle, Q[b], K[b], V[b], u[b], dO[b], k, w,
                                                   "hard", "soft")
        assert rel_err(res["o"][b], o) < 1e-10
        assert rel_err(res["dk"][b], dk) < 1e-9
        assert rel_err(res["du"][b], gu) < 1e-8


SEL_LONG = [(kind, 16384, 1024.0, 512) for kind in ("recency", "iid", "ties", "constant")] + [
    # wide tau bands: the segmented large-cap pass and its global-scratch overflow
    ("iid", 32768, 4096.0, 64),
    ("iid", 12000, 300.5, 700),
]


@pytest.mark.parametrize("kind,L,k,w", SEL_LONG, ids=[f"{c[0]}-{c[1]}-{c[2]}" for c in SEL_LONG])
def test_selection_long_sequence(cuda, oracle, kind, L, k, w):
    """cfg3-length sequence: retention intervals and tau against the oracle's
    heap restatement (bit-exact sets; tau 1e-9 on non-degenerate steps)."""
    import torch

    from paper_2406_16747_b200 import ops

    rng = np.random.default_rng(99)
    u = _scores(rng, L, kind)
    cfg = ops.AttnConfig(k=k, window=w)
    sel = ops.select(torch.from_numpy(u)[None].to(cuda), cfg)
    leave = sel.leave[0].cpu().numpy()
    tau = sel.tau[0].cpu().numpy()
    T = L - w
    # reference tau from the heap stream restatement
    tau_ref, _ = oracle.stream_taus(u[:T], k)
    # retention: size min(t+1, floor k) and membership = top-floor(k) of the prefix
    kf = int(np.floor(k))
    order = np.lexsort((np.arange(T), -u[:T]))  # value desc, index asc
    rank_pos = np.empty(T, np.int64)
    rank_pos[order] = np.arange(T)
    for t in (0, 1, kf - 2, kf - 1, kf, kf + 1, T // 3, T // 2, T - 2, T - 1):
        if t < 0 or t >= T:
            continue
        members = np.nonzero((np.arange(T) <= t) & (leave[:T] > t))[0]
        pref = np.arange(t + 1)
        best = pref[np.lexsort((pref, -u[: t + 1]))][: min(kf, t + 1)]
        np.testing.assert_array_equal(members, np.sort(best))
    # tau
    fin = np.isfinite(tau_ref)
    np.testing.assert_array_equal(np.isfinite(tau[:T]), fin)
    csum_ok = 0
    for t in np.nonzero(fin)[0][:: max(1, fin.sum() // 2000)]:
        f = u[: t + 1] - tau_ref[t]
        if np.any((f > 0) & (f < 1)):
            assert abs(tau[t] - tau_ref[t]) <= 1e-9 * max(1.0, abs(tau_ref[t])), t
            csum_ok += 1
    assert np.all(np.diff(tau[:T][fin]) >= 0)


TC_CASES = [
    # L, H, p, k, w, key, mask, kind
    (1024, 2, 128, 64.0, 64, "hard", "soft", "recency"),
    (1000, 2, 128, 100.5, 200, "hard", "soft", "iid"),
    (777, 3, 64, 50.0, 33, "soft", "soft", "iid"),
    (640, 1, 128, 24.0, 128, "hard", "straight_through", "ties"),
    (513, 2, 64, 300.0, 1, "hard", "soft", "recency"),
    (384, 2, 128, 16.0, 300, "soft", "straight_through", "falling"),
    (100, 1, 64, 8.0, 7, "hard", "soft", "constant"),
    (2048, 2, 128, 256.0, 256, "hard", "soft", "recency"),
]


@pytest.mark.parametrize("case", TC_CASES, ids=[str(c) for c in TC_CASES])
def test_tensor_core_path_vs_oracle(cuda, oracle, case):
    """BF16 tcgen05 kernels against the oracle on the bf16-rounded inputs (2e-2),
    and against the CUDA-core gather path on the same inputs."""
    import torch

    L, H, p, k, w, km, mm, kind = case
    rng = np.random.default_rng(L + 13 * H + p)
    rnd = lambda a: torch.from_numpy(a).to(torch.bfloat16).double().numpy()
    Q, K, V, dO = (rnd(rng.normal(size=(L, H, p))) for _ in range(4))
    u = _scores(rng, L, kind)
    sel, o, lse, dq, dk, dv, gu = _oracle_core(oracle, Q, K, V, u, dO, k, w, km, mm)
    tc = run_core_gpu(Q, K, V, u, dO, k=k, w=w, key_mode=km, mask_mode=mm, dtype="bf16")
    ga = run_core_gpu(Q, K, V, u, dO, k=k, w=w, key_mode=km, mask_mode=mm, dtype="bf16",
                      force_gather=True)
    for name, ref in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert rel_err(tc[name], ref) < 2e-2, (name, rel_err(tc[name], ref))
        assert rel_err(tc[name], ga[name]) < 2e-2, (name, rel_err(tc[name], ga[name]))
    np.testing.assert_allclose(tc["lse"], lse.T, rtol=0, atol=2e-2)
    if np.abs(gu).max() > 0:
        assert rel_err(tc["du"], gu) < 2e-2, rel_err(tc["du"], gu)


FULL_CASES = [
    # BASELINE.json configs at full size, one sequence each: (L, H, p, k, w)
    ("cfg3", 16384, 32, 128, 1024.0, 512),
    ("cfg2", 4096, 12, 64, 256.0, 256),
]


@pytest.mark.parametrize("case", FULL_CASES, ids=[c[0] for c in FULL_CASES])
@pytest.mark.parametrize("kind", ["recency", "iid"])
def test_full_size_tensor_core_path(cuda, oracle, case, kind):
    """Full BASELINE shapes, bf16 tcgen05 path, two independent checks:
    (1) sampled query rows recomputed in float64 from the C oracle's selection
        (Sel_i, tau_i) — o_i and dq_i within 2e-2;
    (2) every output against the f32 CUDA-core gather path on the same
        (bf16-rounded) inputs — o, dq, dk, dv and du within 2e-2."""
    import torch

    from paper_2406_16747_b200 import ops

    name, L, H, p, k, w = case
    rng = np.random.default_rng(L + H)
    g = torch.Generator(device=cuda)
    g.manual_seed(L)
    shape = (1, L, H, p)
    q, kk, v, do = (torch.randn(shape, generator=g, device=cuda).to(torch.bfloat16) for _ in range(4))
    u_np = _scores(rng, L, kind)
    u = torch.from_numpy(u_np)[None].to(cuda)
    cfg = ops.AttnConfig(k=k, window=w)
    o, lse, sel = ops.attn_fwd(q, kk, v, u, cfg)
    dq, dk, dv, du = ops.attn_bwd(q, kk, v, o, do, lse, u, sel, cfg)
    gcfg = ops.AttnConfig(k=k, window=w, force_gather=True)
    f = lambda t: t.float().contiguous()
    og, lseg, selg = ops.attn_fwd(f(q), f(kk), f(v), u, gcfg)
    dqg, dkg, dvg, dug = ops.attn_bwd(f(q), f(kk), f(v), og, f(do), lseg, u, selg, gcfg)
    torch.cuda.synchronize()
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))
    for nm, a, b_ in (("o", o, og), ("dq", dq, dqg), ("dk", dk, dkg), ("dv", dv, dvg)):
        assert rel(a, b_) < 2e-2, (nm, rel(a, b_))
    assert rel(du, dug) < 2e-2, rel(du, dug)
    # (1) sampled rows against the oracle's selection
    osel = oracle.select(u_np, k, w)
    Qn, Kn, Vn, dOn = (t[0].double().cpu().numpy() for t in (q, kk, v, do))
    on, dqn = o[0].double().cpu().numpy(), dq[0].double().cpu().numpy()
    scale = 1.0 / np.sqrt(p)
    rows = np.unique(np.concatenate([[0, w - 1, w, w + int(k), L - 1], rng.integers(0, L, size=40)]))
    num_o = den_o = num_q = den_q = 0.0
    for i in rows:
        att = osel.att_of(i)
        ns = osel.n_sel[i]
        gates = np.ones(len(att))
        gates[:ns] = np.clip(u_np[att[:ns]] - osel.tau_q[i], 0, 1)
        for h in range(H):
            a = scale * Kn[att, h] @ Qn[i, h]
            P = np.exp(a - a.max())
            P /= P.sum()
            oo = (P * gates) @ Vn[att, h]
            dP = Vn[att, h] @ dOn[i, h]
            dlt = np.sum(P * gates * dP)
            dqq = scale * ((P * (gates * dP - dlt)) @ Kn[att, h])
            num_o += np.sum((on[i, h] - oo) ** 2)
            den_o += np.sum(oo ** 2)
            num_q += np.sum((dqn[i, h] - dqq) ** 2)
            den_q += np.sum(dqq ** 2)
    assert np.sqrt(num_o / den_o) < 2e-2, np.sqrt(num_o / den_o)
    assert np.sqrt(num_q / den_q) < 2e-2, np.sqrt(num_q / den_q)


@pytest.mark.parametrize("cap", ["", "3"])
def test_fused_dq_backward_opt_in(cuda, cap):
    """The opt-in fused-dQ backward (SKB_BWD_FUSEDQ=1: dQ^T = K^T dS^T in the
    key-major passes, fp32 reductions) against the gather path, including
    capped persistent grids (every cross-item ring and the dQ^T read-back wrap)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, SKB_BWD_FUSEDQ="1")
    if cap:
        env["SKB_MAX_CTAS"] = cap
    r = subprocess.run([sys.executable, os.path.join(here, "scripts", "persist_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("uni", ["0", "1", "q96", "q128"])
def test_unified_and_two_pass_key_major_backward(cuda, uni):
    """Dense sequences take the unified key-major pass (window + selection of a
    contiguous key tile in one kernel, SKB_BWD_UNI=1, the default); SKB_BWD_UNI=0
    keeps the selected + window passes with bf16 partials; SKB_BWD_QTILE=96/128
    runs the unified pass with taller query tiles. All against the
    gather path, with capped persistent grids so every ring wraps (the recency
    cases are dense, the iid ones sparse, the chunked one never unified)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, SKB_MAX_CTAS="5")
    if uni.startswith("q"):  # the unified pass with 96- / 128-query tiles (k_bwd_kmaj_q, opt-in)
        env.update(SKB_BWD_UNI="1", SKB_BWD_QTILE=uni[1:])
    else:
        env["SKB_BWD_UNI"] = uni
    r = subprocess.run([sys.executable, os.path.join(here, "scripts", "persist_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("cap", ["2", "7"])
def test_persistent_grids_many_items_per_cta(cuda, cap):
    """The persistent kernels with their grid capped (SKB_MAX_CTAS): each CTA
    walks dozens of work items, so every cross-item ring (K/V, Q/dO, S, the
    accumulators, the partial and staging buffers) wraps many times; results
    must match the gather path as with one item per CTA."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, SKB_MAX_CTAS=cap)
    r = subprocess.run([sys.executable, os.path.join(here, "scripts", "persist_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_persistent_grid_size_never_changes_a_bit(cuda, tmp_path):
    """Forward and backward outputs (o, lse, dq, dk, dv) are bit-identical with
    one CTA, three CTAs and the full persistent grid: no cross-item ring state
    leaks between work items."""
    import os
    import subprocess
    import sys

    import torch

    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for cap in ("0", "1", "3"):
        f = tmp_path / f"out{cap}.pt"
        env = dict(os.environ, SKB_MAX_CTAS=cap)
        r = subprocess.run([sys.executable, os.path.join(here, "scripts", "fwd_det.py"), str(f)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(torch.load(f))
    for other in outs[1:]:
        for kind in outs[0]:
            for nm, x, y in zip(("o", "lse", "dq", "dk", "dv"), outs[0][kind], other[kind]):
                assert torch.equal(x, y), (kind, nm)
