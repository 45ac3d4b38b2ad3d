"""GPU: the operator helpers around the attention path, each against the
compiled reference (oracle/_ref) on the same inputs.

  * Stream.push's StreamStepResult — tau, t, inserted and the evicted list —
    per push, fresh and after a deserialize (proj/src/stream.cpp:72-152,
    proj/tests/test_stream.cpp:28-62,139-163);
  * stream_mask / SelectionMask (proj/src/stream.cpp:199-222,
    proj/tests/test_stream.cpp:177-200) and StreamState::solution;
  * sparsek_partial + PartialSortStats (proj/src/sparsek_op.cpp:116-139,
    proj/tests/test_sparsek_op.cpp:228-255) and sparsek_st (:167-172, :265-274);
  * dense_causal_attention and its backward (proj/src/attention.cpp:76-205);
  * AttnTape + sparsek_attention_backward from the tape (attention.hpp:47-91).
"""
import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _z(rng, n, kind):
    if kind == "normal":
        return rng.normal(size=n)
    if kind == "ties":
        return 0.5 * rng.integers(-3, 4, size=n).astype(np.float64)
    if kind == "rising":
        return rng.normal(size=n) + 0.02 * np.arange(n)
    if kind == "falling":
        return -0.05 * np.arange(n) + 0.2 * rng.normal(size=n)
    raise ValueError(kind)


STREAM_CASES = [("normal", 3.5, 0), ("ties", 6.0, 0), ("rising", 10.0, 0), ("falling", 4.0, 0),
                ("normal", 5.0, 12), ("ties", 2.0, 3)]


@pytest.mark.parametrize("kind,k,heap_cap", STREAM_CASES)
def test_stream_push_events_vs_reference(cuda, reference, kind, k, heap_cap):
    from paper_2406_16747_b200 import Stream

    rng = np.random.default_rng(hash((kind, k)) & 0xFFFF)
    z = _z(rng, 400, kind)
    tau_r, ins_r, _, ev_r = reference.stream_events(z, k, heap_cap)
    s = Stream(k, heap_cap=heap_cap, capacity=1024)
    for t in range(len(z)):
        r = s.push(z[t])
        assert r["t"] == t + 1
        assert r["inserted"] == ins_r[t], t
        assert r["evicted"] == ev_r[t], (t, r["evicted"], ev_r[t])
        if np.isfinite(tau_r[t]):
            assert r["tau"] == tau_r[t], t  # identical push/scan arithmetic
        else:
            assert r["tau"] is None


@pytest.mark.parametrize("kind", ["normal", "ties"])
def test_stream_events_after_deserialize(cuda, reference, kind):
    """After a blob round trip the first push reports only what it evicts
    (the advisor's finding: no replay of earlier evictions)."""
    from paper_2406_16747_b200 import Stream

    rng = np.random.default_rng(7)
    z = _z(rng, 300, kind)
    k, cut = 8.0, 150
    _, _, _, ev_r = reference.stream_events(z, k)
    for blob in (reference.stream_blob(z[:cut], k), None):
        if blob is None:  # our own blob
            s0 = Stream(k, capacity=512)
            for v in z[:cut]:
                s0.push(v)
            blob = s0.serialize()
        s = Stream.deserialize(blob, capacity=512)
        for t in range(cut, len(z)):
            assert s.push(z[t])["evicted"] == ev_r[t], t


@pytest.mark.parametrize("kind,k", [("normal", 5.5), ("ties", 4.0), ("rising", 12.0), ("normal", 50.0)])
def test_stream_mask_and_solution_vs_reference(cuda, reference, kind, k):
    from paper_2406_16747_b200 import Stream, stream_mask

    rng = np.random.default_rng(11)
    z = _z(rng, 120, kind)
    s = Stream(k, capacity=256)
    for n in (3, 30, 120):
        while s.t < n:
            s.push(z[s.t])
        pos, hard, soft, idx = reference.stream_mask(z[:n], k)
        m = stream_mask(s)
        np.testing.assert_array_equal(m.positions, pos)
        np.testing.assert_array_equal(m.hard, hard)
        np.testing.assert_array_equal(m.soft, soft)
        np.testing.assert_array_equal(m.indices, idx)
        sol = s.solution()
        _, _, _, p_last = reference.stream(z[:n], k)
        np.testing.assert_array_equal(sol["p"], p_last)


def test_stream_mask_empty_state_errors(cuda):
    from paper_2406_16747_b200 import ArgumentError, Stream, stream_mask

    with pytest.raises(ArgumentError):
        stream_mask(Stream(2.0))


@pytest.mark.parametrize("kind", ["normal", "ties", "rising"])
def test_sparsek_partial_stats_vs_reference(cuda, reference, kind):
    import paper_2406_16747_b200 as sk

    rng = np.random.default_rng(3)
    stats = sk.PartialSortStats()
    calls = fallbacks = 0
    for trial in range(40):
        m = int(rng.integers(4, 80))
        z = _z(rng, m, kind)
        k = float(rng.integers(1, m)) if trial % 2 else float(rng.uniform(0.5, m - 1))
        cap = int(rng.integers(int(np.ceil(k)), m + 1))
        p_r, tau_r, c, f = reference.sparsek_partial_stats(z, k, cap)
        calls += c
        fallbacks += f
        got = sk.sparsek_partial(z, k, cap, stats)
        np.testing.assert_allclose(got["p"], p_r, rtol=0, atol=1e-12)
    assert (stats.calls, stats.fallbacks) == (calls, fallbacks)
    assert fallbacks > 0  # both branches were exercised
    # the reference's own partial-sort fallback case: 64 constants (test_sparsek_op.cpp:242-250)
    st = sk.PartialSortStats()
    r = sk.sparsek_partial(np.full(64, 0.5), 8.0, 8, st)
    np.testing.assert_allclose(r["p"], np.full(64, 8.0 / 64), atol=1e-12)
    assert (st.calls, st.fallbacks) == (1, 1)


def test_sparsek_st_vs_reference(cuda, reference):
    import paper_2406_16747_b200 as sk

    rng = np.random.default_rng(5)
    for kind in ("normal", "ties"):
        z = _z(rng, 50, kind)
        for k in (1.0, 3.5, 17.0):
            fwd_r, p_r = reference.sparsek_st(z, k)
            got = sk.sparsek_st(z, k)
            np.testing.assert_array_equal(got["forward"], fwd_r)
            np.testing.assert_allclose(got["backward_carrier"]["p"], p_r, rtol=0, atol=1e-12)


@pytest.mark.parametrize("L,D,H", [(64, 16, 2), (200, 32, 4), (129, 24, 3)])
def test_dense_attention_and_backward_vs_reference(cuda, reference, L, D, H):
    import paper_2406_16747_b200 as sk

    rng = np.random.default_rng(L + D)
    x = rng.normal(size=(L, D))
    ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
    g = rng.normal(size=(L, D))
    y_ref, gr = reference.dense_attention_grads(x, *ws, g, heads=H)
    np.testing.assert_allclose(reference.dense_attention(x, *ws, heads=H), y_ref, rtol=0, atol=1e-12)
    assert rel_err(sk.dense_attention(x, *ws, heads=H), y_ref) < 1e-10
    y, grads = sk.dense_attention_grads(x, *ws, g, heads=H)
    assert rel_err(y, y_ref) < 1e-10
    for name in ("dx", "dwq", "dwk", "dwv", "dwo"):
        assert rel_err(grads[name], gr[name]) < 1e-9, (name, rel_err(grads[name], gr[name]))


@pytest.mark.parametrize("km,mm,chunk", [("hard", "soft", 0), ("soft", "straight_through", 0), ("hard", "soft", 48)])
def test_tape_forward_backward_vs_reference(cuda, reference, km, mm, chunk):
    """sparsek_attention with a tape, then sparsek_attention_backward from it:
    tape fields (q, k, v, head_concat, raw, u, tau_push, per-query attended
    lists and gates) and AttnGrads against the reference's tape run."""
    from oracle.oracle import ref_cfg

    import paper_2406_16747_b200 as sk

    L, D, H, k, w = 160, 24, 3, 12.5, 10
    rng = np.random.default_rng(17)
    x = rng.normal(size=(L, D))
    ws = [rng.normal(size=(D, D)) * 0.6 / np.sqrt(D) for _ in range(4)]
    wsc = rng.normal(size=D) / np.sqrt(D)
    g = rng.normal(size=(L, D))
    cfg = ref_cfg(k, w, heads=H, key_mode=km, mask_mode=mm)
    tape_r, gr = reference.attention(x, *ws, wsc, cfg, grad_out=g, chunk_len=chunk)
    y, tape = sk.attention_with_tape(x, *ws, wsc, k, w, heads=H, key_mode=km, mask_mode=mm, chunk_len=chunk)
    assert rel_err(y, tape_r.y) < 1e-10
    for name in ("q", "k", "v"):
        got = getattr(tape, name)[0].reshape(L, D).cpu().numpy()
        assert rel_err(got, getattr(tape_r, name)) < 1e-12, name
    assert rel_err(tape.head_concat[0].reshape(L, D).cpu().numpy(), tape_r.head_concat) < 1e-10
    np.testing.assert_array_equal(tape.u[0].cpu().numpy(), tape_r.u)
    np.testing.assert_array_equal(tape.raw[0].cpu().numpy(), tape_r.raw)
    tp = tape.tau_push
    fin = np.isfinite(tape_r.tau_push)
    np.testing.assert_array_equal(np.isfinite(tp), fin)
    np.testing.assert_allclose(tp[fin], tape_r.tau_push[fin], rtol=1e-9, atol=1e-12)
    recs = tape.queries()
    for i in range(L):
        a0, a1 = tape_r.att_off[i], tape_r.att_off[i + 1]
        np.testing.assert_array_equal(recs[i].att, tape_r.att[a0:a1])
        assert recs[i].n_sel == tape_r.n_sel[i]
    grads = sk.attention_backward(tape, g)
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dw_score"):
        assert rel_err(grads[name], gr[name]) < 1e-8, (name, rel_err(grads[name], gr[name]))
