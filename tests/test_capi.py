"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and
rejects bad configurations before touching the GPU (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparsek_b200.h")
LIB = os.path.join(ROOT, "paper_2406_16747_b200", "libsparsek_b200.so")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:const char\*|int|skb_\w+\*)\s+(skb_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("skb_select", "skb_attn_fwd", "skb_attn_bwd", "skb_score_fwd", "skb_score_bwd",
                 "skb_sparsek", "skb_sparsek_jvp", "skb_topk_hard", "skb_cache_create",
                 "skb_cache_step", "skb_stream_push", "skb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libsparsek_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_loader_binds_all_declared():
    from paper_2406_16747_b200 import _lib

    assert set(declared()) == set(_lib.exported_symbols())
    lib = _lib.load()
    assert lib.skb_version() == 1


def test_config_errors_map_to_reference_taxonomy():
    """ConfigError before any compute (proj/src/attention.cpp:15-35) -> ValueError."""
    from paper_2406_16747_b200 import _lib
    from paper_2406_16747_b200.ops import AttnConfig, make_desc
    import torch

    lib = _lib.load()
    lay = _lib.SelectLayout()
    bad = make_desc(1, 16, 1, 8, AttnConfig(k=0.5, window=0), torch.float32)
    rc = lib.skb_select_layout_of(bad, lay)
    assert rc == 4  # SKB_ECONFIG
    with pytest.raises(ValueError):
        _lib.check(rc)
    bad2 = make_desc(1, 16, 1, 8, AttnConfig(k=-1.0, window=2), torch.float32)
    with pytest.raises(_lib.ConfigError):
        _lib.check(lib.skb_select_layout_of(bad2, lay))
    ok = make_desc(2, 300, 2, 8, AttnConfig(k=8.5, window=8), torch.float32)
    _lib.check(lib.skb_select_layout_of(ok, lay))
    assert lay.qb_cap == 256 and lay.nqb == 3 and lay.total_bytes > 0  # floor(k)+128 rounded to 128


def test_error_classes_follow_pybind_mapping():
    import paper_2406_16747_b200 as s

    assert issubclass(s.ShapeError, ValueError)
    assert issubclass(s.ArgumentError, ValueError)
    assert issubclass(s.ConfigError, ValueError)
    assert issubclass(s.NumericError, ArithmeticError)
