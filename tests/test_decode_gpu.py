"""GPU: K5, the constant-(floor(k)+w) decode cache (skb_cache_*), and the
device-resident stream (skb_stream_*).

Properties ported from the reference's own tests:
  * decode is the batch forward, one row at a time
    (proj/tests/test_cache.cpp:128-149) — checked against the C oracle's
    batch forward on the same inputs;
  * retained rows = brute-force top-floor(k) + window
    (proj/tests/test_cache.cpp:84-97) and peak_kv <= floor(k)+w+1
    (proj/tests/test_cache.cpp:124,148; proj/tests/acceptance.cpp:538-543);
  * the stream's tau equals the reference StreamState's bit for bit
    (proj/tests/test_stream.cpp:28-62), rejections are permanent (:85-97).
Tolerances: float64 1e-9 (float64 pools accumulate in float64), float32 1e-5 relative, bfloat16 2e-2 (decode accumulates in fp32).
"""
import math

import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _scores(rng, L, kind):
    if kind == "recency":
        return rng.normal(size=L) + 0.01 * np.arange(1, L + 1)
    if kind == "iid":
        return rng.normal(size=L)
    if kind == "ties":
        return 0.5 * rng.integers(-4, 5, size=L).astype(np.float64)
    if kind == "constant":
        return np.full(L, 0.25)
    raise ValueError(kind)


CASES = [
    # B, L, H, p, k, w, key, mask, kind, prompt
    (2, 300, 2, 16, 12.5, 8, "hard", "soft", "recency", 0),
    (3, 260, 2, 32, 20.0, 16, "soft", "soft", "iid", 100),
    (1, 200, 1, 64, 9.0, 0, "hard", "straight_through", "ties", 37),
    (2, 150, 2, 32, 0.0, 12, "hard", "soft", "iid", 20),        # pure window
    (2, 120, 2, 32, 0.5, 6, "soft", "soft", "iid", 0),          # floor(k) = 0, stream on
    (1, 90, 4, 128, 7.0, 5, "hard", "soft", "constant", 30),
    (2, 40, 2, 8, 8.0, 64, "hard", "soft", "iid", 10),          # never leaves the window
    # survivor arrays outgrow the control kernel's shared-memory staging
    # (4096 entries) part-way: both the staged and the global-array push
    (1, 4600, 1, 16, 4300.0, 8, "hard", "soft", "recency", 200),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[:9]) for c in CASES])
@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_decode_equals_batch_forward(cuda, oracle, case, dtype):
    import torch

    from paper_2406_16747_b200 import ops

    B, L, H, p, k, w, km, mm, kind, prompt = case
    rng = np.random.default_rng(B * 1000 + L)
    Q, K, V = (rng.normal(size=(B, L, H, p)) for _ in range(3))
    U = np.stack([_scores(rng, L, kind) for _ in range(B)])
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    if dtype == "bf16":
        rnd = lambda a: torch.from_numpy(a).to(torch.bfloat16).double().numpy()
        Q, K, V = rnd(Q), rnd(K), rnd(V)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda).to(tdt)
    cfg = ops.AttnConfig(k=k, window=w, key_mode=km, mask_mode=mm)
    cache = ops.DecodeCache(B, H, p, cfg, max_len=L, dtype=tdt)
    ut = torch.from_numpy(U).to(cuda)
    if prompt:
        cache.prefill(t(K[:, :prompt]), t(V[:, :prompt]), ut[:, :prompt].contiguous())
    outs = []
    for i in range(prompt, L):
        outs.append(cache.step(t(Q[:, i]), t(K[:, i]), t(V[:, i]), ut[:, i].contiguous()))
    got = torch.stack(outs, 1).double().cpu().numpy()  # [B, L - prompt, H, p]
    tol = {"f64": 1e-9, "f32": 1e-5, "bf16": 2e-2}[dtype]
    kf = int(math.floor(k))
    for b in range(B):
        sel = oracle.select(U[b], k, w)
        o, _, _ = oracle.attn_fwd(Q[b], K[b], V[b], sel, kbudget=k, window=w, key_mode=km,
                                  mask_mode=mm)
        assert rel_err(got[b], o[prompt:]) < tol, (b, rel_err(got[b], o[prompt:]))
        st = cache.state(b)
        assert st["seen"] == L
        # retained rows after the last step = what the last query read
        att = sel.att_of(L - 1)
        expect = sorted(att[: sel.n_sel[L - 1]]) + sorted(att[sel.n_sel[L - 1]:]) if w > 0 \
            else sorted(att[: sel.n_sel[L - 1]])
        np.testing.assert_array_equal(st["positions"], np.asarray(expect, np.int64))
        assert st["peak"] <= kf + w + 1
        if L > kf + w + 1:
            assert st["peak"] == kf + w + 1 or kf == 0


def test_decode_retention_every_step(cuda, oracle):
    """Brute-force top-floor(k) + window after every step (test_cache.cpp:66-126)."""
    import torch

    from paper_2406_16747_b200 import ops

    L, H, p, k, w = 160, 1, 8, 6.0, 4
    rng = np.random.default_rng(9)
    u = 0.5 * rng.integers(-3, 4, size=L).astype(np.float64)  # heavy ties
    cfg = ops.AttnConfig(k=k, window=w)
    cache = ops.DecodeCache(1, H, p, cfg, max_len=L, dtype=torch.float32)
    z = torch.zeros((1, H, p), dtype=torch.float32, device=cuda)
    for i in range(L):
        cache.step(z, z, z, torch.tensor([u[i]], dtype=torch.float64, device=cuda))
        t = i - w  # pushes so far: positions 0..t
        if t >= 0:
            order = sorted(range(t + 1), key=lambda j: (-u[j], j))[: int(k)]
            sel = sorted(order)
        else:
            sel = []
        win = list(range(max(0, i - w + 1), i + 1))
        assert list(cache.state(0)["positions"]) == sel + win, i


def test_decode_tau_bit_exact_vs_reference_stream(cuda, reference):
    import torch

    from paper_2406_16747_b200 import ops

    L, k, w = 500, 17.5, 9
    rng = np.random.default_rng(2)
    u = rng.normal(size=L)
    cache = ops.DecodeCache(1, 1, 8, ops.AttnConfig(k=k, window=w), max_len=L, dtype=torch.float32)
    taus = []
    z = torch.zeros((1, 1, 8), dtype=torch.float32, device=cuda)
    for i in range(L):
        cache.step(z, z, z, torch.tensor([u[i]], dtype=torch.float64, device=cuda))
        taus.append(cache.state(0)["tau"])
    tau_ref, _, _, _ = reference.stream(u[: L - w], k)
    got = np.asarray(taus[w:])
    np.testing.assert_array_equal(got, tau_ref)  # identical push/scan arithmetic


def test_prefill_then_step_matches_step_only(cuda):
    import torch

    from paper_2406_16747_b200 import ops

    B, L, H, p, k, w, P = 2, 220, 2, 64, 30.0, 17, 150
    rng = np.random.default_rng(4)
    Q, K, V = (torch.from_numpy(rng.normal(size=(B, L, H, p))).to(cuda).to(torch.bfloat16)
               for _ in range(3))
    U = torch.from_numpy(rng.normal(size=(B, L)) + 0.01 * np.arange(L)).to(cuda)
    cfg = ops.AttnConfig(k=k, window=w)
    a = ops.DecodeCache(B, H, p, cfg, max_len=L)
    b = ops.DecodeCache(B, H, p, cfg, max_len=L)
    a.prefill(K[:, :P].contiguous(), V[:, :P].contiguous(), U[:, :P].contiguous())
    for i in range(P):
        b.step(Q[:, i].contiguous(), K[:, i].contiguous(), V[:, i].contiguous(), U[:, i].contiguous())
    for i in range(P, L):
        args = (Q[:, i].contiguous(), K[:, i].contiguous(), V[:, i].contiguous(), U[:, i].contiguous())
        oa, ob = a.step(*args), b.step(*args)
        assert torch.equal(oa, ob), i
    for s in range(B):
        sa, sb = a.state(s), b.state(s)
        np.testing.assert_array_equal(sa["positions"], sb["positions"])
        assert sa["tau"] == sb["tau"] and sa["peak"] == sb["peak"]


def test_decode_errors(cuda):
    import torch

    from paper_2406_16747_b200 import ops
    from paper_2406_16747_b200._lib import ShapeError

    cache = ops.DecodeCache(1, 1, 8, ops.AttnConfig(k=2.0, window=2), max_len=3,
                            dtype=torch.float32)
    z = torch.zeros((1, 1, 8), dtype=torch.float32, device=cuda)
    u = torch.zeros(1, dtype=torch.float64, device=cuda)
    with pytest.raises(ShapeError):
        cache.step(torch.zeros((1, 2, 8), dtype=torch.float32, device=cuda), z, z, u)
    for _ in range(3):
        cache.step(z, z, z, u)
    cache.step(z, z, z, u)  # the 4th position overflows seq_len: reported by state()
    with pytest.raises(ShapeError):
        cache.state(0)


# ------------------------------------------------------------------ stream

@pytest.mark.parametrize("kind", ["iid", "ties", "constant", "recency"])
@pytest.mark.parametrize("k", [1.0, 3.5, 16.0])
def test_stream_matches_reference(cuda, reference, kind, k):
    import paper_2406_16747_b200 as sparsek

    rng = np.random.default_rng(13)
    z = _scores(rng, 120, kind)
    tau_ref, ins_ref, surv_ref, _ = reference.stream(z, k)
    st = sparsek.Stream(k)
    for i in range(len(z)):
        r = st.push(z[i])
        tr = tau_ref[i]
        assert (r["tau"] is None) == (not math.isfinite(tr))
        if r["tau"] is not None:
            assert r["tau"] == tr, i  # bit-identical
        assert r["inserted"] == bool(ins_ref[i])
        assert st.survivors == surv_ref[i]


def test_stream_rejection_is_permanent(cuda):
    import paper_2406_16747_b200 as sparsek

    st = sparsek.Stream(2.0)
    for z in (0.9, 0.5, 0.1, 2.0, 3.0):
        st.push(z)
    tau = st.tau
    r = st.push(tau - 0.5)
    assert not r["inserted"] and st.is_evicted(st.t - 1)
    sol = st.solution()
    assert sol["p"][st.t - 1] == 0.0


@pytest.mark.parametrize("kind", ["iid", "ties", "recency"])
def test_stream_wire_format_interop(cuda, reference, kind):
    """The device stream speaks the reference's StreamState wire format
    (proj/src/stream.cpp:224-289) both ways, and resuming from a blob gives the
    same taus as never stopping (bit for bit)."""
    import paper_2406_16747_b200 as sparsek

    rng = np.random.default_rng(21)
    z = _scores(rng, 300, kind)
    k, n1 = 7.5, 180
    tau_all, _, _, _ = reference.stream(z, k)
    # ours -> reference
    st = sparsek.Stream(k)
    for x in z[:n1]:
        st.push(x)
    blob = st.serialize()
    tau_ref_resumed = reference.stream_resume(blob, z[n1:])
    np.testing.assert_array_equal(tau_ref_resumed, tau_all[n1:])
    # reference -> ours
    st2 = sparsek.Stream.deserialize(reference.stream_blob(z[:n1], k))
    got = []
    for x in z[n1:]:
        r = st2.push(x)
        got.append(r["tau"] if r["tau"] is not None else -np.inf)
    np.testing.assert_array_equal(np.asarray(got), tau_all[n1:])
    # ours -> ours
    st3 = sparsek.Stream.deserialize(blob)
    got3 = [st3.push(x)["tau"] for x in z[n1:]]
    np.testing.assert_array_equal(np.asarray(got3, dtype=float), tau_all[n1:])
