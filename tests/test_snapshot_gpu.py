"""GPU: decode-state snapshots in the reference's SparseKvCache format
(serialize / deserialize, proj/src/cache.cpp:416-545; save/load_cache_snapshot
file framing :579-618), against the C reference build (oracle/_ref):
  * ours -> reference: the reference resumes from our payload and generates
    the same rows as an uninterrupted reference run;
  * reference -> ours: we resume from the reference's payload likewise;
  * every non-row field of our payload (scores, norm state, stream, ring, cache
    heap in the reference's array order, evicted bitmap, pending evictions,
    peak) equals the reference's byte for byte; rows agree to float64 rounding;
  * ours -> ours at the q/k/v level resumes bit-identically (bf16 and f32)."""
import struct

import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def parse(blob):
    """Field-wise view of a SparseKvCache::serialize payload."""
    off = 0

    def u64():
        nonlocal off
        v = struct.unpack_from("<Q", blob, off)[0]
        off += 8
        return v

    def f64():
        nonlocal off
        v = struct.unpack_from("<d", blob, off)[0]
        off += 8
        return v

    def u8():
        nonlocal off
        v = blob[off]
        off += 1
        return v

    f = {"d_model": u64(), "heads": u64(), "window": u64(), "cap": u64(), "k": f64(), "lin": u8(),
         "has_stream": u8(), "t": u64()}
    f["scores"] = [f64() for _ in range(u64())]
    f["norm"] = (u64(), f64(), f64(), f64())
    if f["has_stream"]:
        n = u64()
        f["stream"] = blob[off:off + n]
        off += n
    f["ring"] = [u64() for _ in range(u64())]
    f["heap"] = [(f64(), u64()) for _ in range(u64())]
    f["cache_pos"] = [u64() for _ in range(u64())]
    rows = []
    D = f["d_model"]
    for _ in range(u64()):
        pos = u64()
        kv = struct.unpack_from(f"<{2 * D}d", blob, off)
        off += 16 * D
        rows.append((pos, np.array(kv)))
    f["rows"] = rows
    nbits = u64()
    f["evicted"] = (nbits, blob[off:off + (nbits + 7) // 8])
    off += (nbits + 7) // 8
    f["pending"] = [u64() for _ in range(u64())]
    f["peak"] = u64()
    assert off == len(blob)
    return f


def _problem(seed, L, D):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(L, D))
    ws = [rng.normal(size=(D, D)) / np.sqrt(D) for _ in range(4)]
    return x, ws, rng.normal(size=D)


CASES = [  # L, D, heads, k, w, prompt, cut
    (120, 32, 2, 10.5, 8, 30, 70),
    (100, 32, 4, 6.0, 0, 0, 45),
    (90, 64, 2, 20.0, 16, 40, 41),
    (80, 32, 2, 0.0, 12, 10, 50),  # no budget: no stream, every departing row dropped
]


def _session(cuda, ws, wsc, H, k, w, L):
    import torch

    from paper_2406_16747_b200 import DecodeSession, ops

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    return DecodeSession(*(t(a) for a in ws), t(wsc), ops.AttnConfig(k=k, window=w), H, batch=1, max_len=L), t


def _run(s, t, x, prompt, lo, hi):
    ys = []
    if prompt and lo == 0:
        ys.append(s.prefill(t(x[None, :prompt]))[0].cpu().numpy())
        lo = prompt
    for i in range(lo, hi):
        ys.append(s.step(t(x[i][None]))[0][None].cpu().numpy())
    return np.concatenate(ys, 0) if ys else np.zeros((0, x.shape[1]))


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_snapshot_interop_with_reference(cuda, reference, case, tmp_path):
    from oracle.oracle import ref_cfg
    from paper_2406_16747_b200.api import load_cache_snapshot, save_cache_snapshot

    L, D, H, k, w, prompt, cut = case
    x, ws, wsc = _problem(L + D, L, D)
    cfg = ref_cfg(k, w, heads=H)
    y_all, _ = reference.decode(x, *ws, wsc, cfg, prompt)
    _, ref_blob = reference.cache_blob(x[:cut], *ws, wsc, cfg, prompt)
    # ours up to cut, snapshot (through the file framing), reference resumes
    s, t = _session(cuda, ws, wsc, H, k, w, L)
    y_ours = _run(s, t, x, prompt, 0, cut)
    assert rel_err(y_ours, y_all[:cut]) < 1e-9
    blob = s.snapshot()
    path = tmp_path / "c.spkc"
    save_cache_snapshot(path, blob)
    assert load_cache_snapshot(path) == blob
    y_ref_resumed = reference.cache_resume(blob, x[cut:], *ws, wsc, cfg)
    assert rel_err(y_ref_resumed, y_all[cut:]) < 1e-9, rel_err(y_ref_resumed, y_all[cut:])
    # field-wise: identical control state, rows within float64 rounding
    a, b = parse(blob), parse(ref_blob)
    for key in ("d_model", "heads", "window", "cap", "k", "lin", "has_stream", "t", "scores", "norm", "ring",
                "heap", "cache_pos", "evicted", "pending", "peak"):
        assert a[key] == b[key], key
    if k > 0:
        sa, sb = a["stream"], b["stream"]
        assert sa[:24] == sb[:24] and sa[32:72] == sb[32:72]  # k, heap_cap, tau, t, counters
    assert [p for p, _ in a["rows"]] == [p for p, _ in b["rows"]]
    for (_, ra), (_, rb) in zip(a["rows"], b["rows"]):
        assert np.abs(ra - rb).max() <= 1e-12 * max(1.0, np.abs(rb).max())
    # the reference's payload -> ours
    s2, t2 = _session(cuda, ws, wsc, H, k, w, L)
    s2.restore(ref_blob)
    y2 = _run(s2, t2, x, 0, cut, L)
    assert rel_err(y2, y_all[cut:]) < 1e-9, rel_err(y2, y_all[cut:])


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_snapshot_resume_is_bit_identical(cuda, dtype):
    import torch

    from paper_2406_16747_b200 import ops

    B, L, H, p, k, w, cut = 2, 200, 2, 64, 30.5, 17, 120
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    Q, K, V = (torch.randn((B, L, H, p), generator=g, device=cuda).to(tdt) for _ in range(3))
    U = torch.randn((B, L), generator=g, device=cuda, dtype=torch.float64) + 0.01 * torch.arange(
        L, device=cuda, dtype=torch.float64)
    cfg = ops.AttnConfig(k=k, window=w)
    a = ops.DecodeCache(B, H, p, cfg, max_len=L, dtype=tdt)
    step = lambda c, i: c.step(Q[:, i].contiguous(), K[:, i].contiguous(), V[:, i].contiguous(),
                               U[:, i].contiguous())
    for i in range(cut):
        step(a, i)
    c2 = ops.DecodeCache(B, H, p, cfg, max_len=L, dtype=tdt)
    for b in range(B):
        c2.restore(a.snapshot(b), b)
        assert a.state(b)["positions"].tolist() == c2.state(b)["positions"].tolist()
    for i in range(cut, L):
        assert torch.equal(step(a, i), step(c2, i)), i
    for b in range(B):  # snapshots after more steps agree too (replay from the restore point)
        assert a.snapshot(b) == c2.snapshot(b)


def test_snapshot_config_mismatch(cuda):
    import torch

    from paper_2406_16747_b200 import ops
    from paper_2406_16747_b200._lib import IoError

    a = ops.DecodeCache(1, 2, 32, ops.AttnConfig(k=8.0, window=4), max_len=50, dtype=torch.float32)
    b = ops.DecodeCache(1, 2, 32, ops.AttnConfig(k=9.0, window=4), max_len=50, dtype=torch.float32)
    with pytest.raises(IoError):
        b.restore(a.snapshot(0))


def test_session_snapshot_per_sequence(cuda):
    """Batched session: every sequence snapshots and restores independently
    (its own scoring state, stream and cache) and resumes bit for bit."""
    import torch

    from paper_2406_16747_b200 import DecodeSession, ops

    B, L, D, H, k, w, prompt, cut = 3, 90, 32, 2, 9.5, 6, 20, 55
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.normal(size=(B, L, D))).to(cuda)
    ws = [torch.from_numpy(rng.normal(size=(D, D)) / np.sqrt(D)).to(cuda) for _ in range(4)]
    wsc = torch.from_numpy(rng.normal(size=D)).to(cuda)
    cfg = ops.AttnConfig(k=k, window=w)
    a = DecodeSession(*ws, wsc, cfg, H, batch=B, max_len=L)
    a.prefill(x[:, :prompt])
    for i in range(prompt, cut):
        a.step(x[:, i])
    b = DecodeSession(*ws, wsc, cfg, H, batch=B, max_len=L)
    for s in (2, 0, 1):  # any order
        b.restore(a.snapshot(s), s)
    assert torch.equal(a.state, b.state)
    for i in range(cut, L):
        assert torch.equal(a.step(x[:, i]), b.step(x[:, i])), i
