"""Loader for the in-tree C-ABI library ``libsparsek_b200.so`` (include/sparsek_b200.h).

There is no fallback: if the library is missing or a call fails, an exception
is raised. Exceptions follow the reference's pybind mapping
(proj/bindings/module.cpp:83-86): Shape/Argument/Config errors are
``ValueError`` subclasses, Numeric errors are ``ArithmeticError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKB_LIB_PATH") or os.path.join(HERE, "libsparsek_b200.so")


class ShapeError(ValueError):
    pass


class ArgumentError(ValueError):
    pass


class ConfigError(ValueError):
    pass


class NumericError(ArithmeticError):
    pass


class IoError(OSError):
    pass


class CudaError(RuntimeError):
    pass


_ERRS = {1: ShapeError, 2: ArgumentError, 3: NumericError, 4: ConfigError, 5: IoError,
         6: CudaError}

SKB_F32, SKB_BF16, SKB_F64 = 0, 1, 2
SKB_FLAG_FORCE_GATHER = 1
SKB_FLAG_LINEAR_MIX = 2


class AttnDesc(C.Structure):
    _fields_ = [("batch", C.c_int64), ("seq_len", C.c_int64), ("heads", C.c_int64),
                ("head_dim", C.c_int64), ("k", C.c_double), ("window", C.c_int64),
                ("scale", C.c_double), ("key_mode", C.c_int32), ("mask_mode", C.c_int32),
                ("dtype", C.c_int32), ("flags", C.c_uint32), ("chunk_len", C.c_int64)]


class Scoring(C.Structure):
    _fields_ = [("norm_mode", C.c_int32), ("slope_order", C.c_int32),
                ("slope_enabled", C.c_int32), ("chunk_len", C.c_int32),
                ("slope_eps", C.c_double)]


class SelectLayout(C.Structure):
    _fields_ = [("leave", C.c_uint64), ("leave_ceil", C.c_uint64), ("tau", C.c_uint64),
                ("nfrac", C.c_uint64), ("qb_count", C.c_uint64), ("qb_list", C.c_uint64),
                ("ever_count", C.c_uint64), ("ever_list", C.c_uint64), ("misc", C.c_uint64),
                ("scratch", C.c_uint64), ("uf", C.c_uint64), ("tauf", C.c_uint64),
                ("qb_leave", C.c_uint64), ("qb_uf", C.c_uint64), ("qb_flags", C.c_uint64),
                ("total_bytes", C.c_uint64), ("qblock", C.c_int64),
                ("nqb", C.c_int64), ("qb_cap", C.c_int64)]


class StreamInfo(C.Structure):
    _fields_ = [("tau", C.c_double), ("t", C.c_int64), ("survivors", C.c_int64),
                ("saturated", C.c_int64), ("cap_drops", C.c_uint64), ("heap_ops", C.c_uint64),
                ("k", C.c_double)]


class XDesc(C.Structure):
    """skb_x_desc: the x-level operator configuration (include/sparsek_b200.h)."""
    _fields_ = [("batch", C.c_int64), ("seq_len", C.c_int64), ("d_model", C.c_int64), ("heads", C.c_int64),
                ("k", C.c_double), ("window", C.c_int64), ("scale", C.c_double), ("key_mode", C.c_int32),
                ("mask_mode", C.c_int32), ("dtype", C.c_int32), ("flags", C.c_uint32), ("chunk_len", C.c_int64),
                ("scoring", Scoring)]


class StreamStep(C.Structure):
    _fields_ = [("tau", C.c_double), ("t", C.c_int64), ("inserted", C.c_int32),
                ("cap_forced", C.c_int32), ("n_evicted", C.c_int64)]


class StreamSolutionInfo(C.Structure):
    _fields_ = [("tau", C.c_double), ("t", C.c_int64), ("n", C.c_int64), ("u_count", C.c_int64),
                ("w_count", C.c_int64), ("degenerate", C.c_int32), ("infeasible", C.c_int32)]


_vp = C.c_void_p
_SIGS = {
    "skb_last_error": ([], C.c_char_p),
    "skb_version": ([], C.c_int),
    "skb_score_fwd": ([C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, C.POINTER(Scoring),
                       _vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_cache_snapshot": ([_vp, C.c_int64, _vp, _vp, C.POINTER(C.c_size_t), _vp], C.c_int),
    "skb_cache_restore": ([_vp, C.c_int64, _vp, C.c_size_t, _vp, _vp], C.c_int),
    "skb_proj_score": ([C.c_int64, C.c_int64, C.c_int64] + [_vp] * 5 + [C.POINTER(Scoring)] + [_vp] * 8,
                       C.c_int),
    "skb_score_raw": ([C.c_int64, C.c_int64, C.c_int32, _vp, _vp, _vp, _vp], C.c_int),
    "skb_score_continue": ([C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, C.POINTER(Scoring),
                            _vp, _vp, _vp, _vp], C.c_int),
    "skb_score_bwd": ([C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, C.POINTER(Scoring),
                       _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_select_layout_of": ([C.POINTER(AttnDesc), C.POINTER(SelectLayout)], C.c_int),
    "skb_select": ([C.POINTER(AttnDesc), _vp, _vp, _vp], C.c_int),
    "skb_attn_fwd": ([C.POINTER(AttnDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_attn_bwd_workspace_size": ([C.POINTER(AttnDesc), C.POINTER(C.c_size_t)], C.c_int),
    "skb_attn_bwd": ([C.POINTER(AttnDesc)] + [_vp] * 14, C.c_int),
    "skb_linmix_phi": ([C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, _vp, _vp], C.c_int),
    "skb_cache_linmix_prefill": ([_vp, _vp, _vp, C.c_int64, _vp], C.c_int),
    "skb_cache_linmix_step": ([_vp] * 9, C.c_int),
    "skb_linmix_workspace_size": ([C.POINTER(AttnDesc), C.POINTER(C.c_size_t)], C.c_int),
    "skb_linmix_fwd": ([C.POINTER(AttnDesc)] + [_vp] * 10, C.c_int),
    "skb_linmix_bwd": ([C.POINTER(AttnDesc)] + [_vp] * 15, C.c_int),
    "skb_sparsek": ([C.c_int64, C.c_int64, _vp, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp],
                    C.c_int),
    "skb_sparsek_jvp": ([C.c_int64, C.c_int64, _vp, C.c_double, _vp, _vp, _vp], C.c_int),
    "skb_topk_hard": ([C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _vp], C.c_int),
    "skb_cache_create": ([C.POINTER(AttnDesc), C.POINTER(_vp)], C.c_int),
    "skb_cache_destroy": ([_vp], C.c_int),
    "skb_cache_step": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_cache_prefill": ([_vp, _vp, _vp, _vp, C.c_int64, _vp], C.c_int),
    "skb_cache_state": ([_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_stream_create": ([C.c_double, C.c_int64, C.c_int64, C.POINTER(_vp)], C.c_int),
    "skb_stream_destroy": ([_vp], C.c_int),
    "skb_stream_push": ([_vp, _vp, C.c_int64, _vp, _vp, _vp], C.c_int),
    "skb_stream_query": ([_vp, C.POINTER(StreamInfo), _vp], C.c_int),
    "skb_support_jvp": ([C.c_int64, _vp, _vp, _vp, _vp], C.c_int),
    "skb_matmul": ([C.c_int32, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp, _vp], C.c_int),
    "skb_xattn_forward": ([C.POINTER(XDesc)] + [_vp] * 7 + [C.POINTER(_vp), _vp], C.c_int),
    "skb_xattn_backward": ([_vp] * 14, C.c_int),
    "skb_xattn_forward_lin": ([C.POINTER(XDesc)] + [_vp] * 8 + [C.POINTER(_vp), _vp], C.c_int),
    "skb_xattn_backward_lin": ([_vp] * 16, C.c_int),
    "skb_xattn_tape_get": ([_vp, C.c_int32, _vp, C.c_size_t, _vp], C.c_int),
    "skb_xattn_destroy": ([_vp], C.c_int),
    "skb_xcache_create": ([C.POINTER(XDesc), C.POINTER(_vp)], C.c_int),
    "skb_xcache_destroy": ([_vp], C.c_int),
    "skb_xcache_forward_chunk": ([_vp, _vp, C.c_int64] + [_vp] * 7, C.c_int),
    "skb_xcache_forward_chunk_lin": ([_vp, _vp, C.c_int64] + [_vp] * 8, C.c_int),
    "skb_xcache_inner": ([_vp], _vp),
    "skb_xcache_norm_state": ([_vp, _vp, C.c_int32, _vp], C.c_int),
    "skb_cache_ledger": ([_vp, C.c_int64, C.c_int32, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, C.c_int64, _vp],
                         C.c_int),
    "skb_stream_push_step": ([_vp, C.c_double, C.POINTER(StreamStep), _vp, C.c_int64, _vp], C.c_int),
    "skb_stream_solution": ([_vp, _vp, _vp, _vp, C.POINTER(StreamSolutionInfo), _vp], C.c_int),
    "skb_stream_survivors": ([_vp, _vp, _vp, _vp, _vp], C.c_int),
    "skb_stream_serialize": ([_vp, _vp, C.POINTER(C.c_size_t), _vp], C.c_int),
    "skb_stream_deserialize": ([_vp, C.c_size_t, C.c_int64, C.POINTER(_vp)], C.c_int),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load libsparsek_b200.so (raises if it is missing — there is no CPU path)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                    "(or __graft_entry__.build()); the SparseK path has no CPU fallback")
            lib = C.CDLL(LIB_PATH)
            for dbg in ("skb_debug_trace", "skb_debug_trace_bwd"):  # -DSKB_TRACE experiment builds
                if hasattr(lib, dbg):
                    getattr(lib, dbg).argtypes = [C.c_void_p, C.c_int]
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int):
    if rc != 0:
        msg = load().skb_last_error().decode(errors="replace")
        raise _ERRS.get(rc, RuntimeError)(msg)


def exported_symbols():
    """Names the header declares (for the load/export test)."""
    return [n for n in _SIGS]
