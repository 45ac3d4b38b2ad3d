"""B200-native SparseK attention (arXiv 2406.16747): the reference's operator
API and Python bindings over hand-written sm_100a kernels.

* Reference-compatible surface (``_sparsek``, proj/bindings/module.cpp):
  ``sparsek, sparsek_jvp, Stream, attention, dense_attention`` and the error
  types — see ``api.py``.
* Torch-level core (device tensors, autograd): ``ops``.
"""
from ._lib import ArgumentError, ConfigError, IoError, NumericError, ShapeError  # noqa: F401
from .api import (  # noqa: F401
    DecodeSession,
    PartialSortStats,
    SelectionMask,
    Stream,
    __version__,
    attention,
    attention_backward,
    attention_grads,
    attention_with_tape,
    chunked_forward,
    dense_attention,
    dense_attention_grads,
    linear_mix_attention,
    linear_mix_attention_grads,
    sparsek,
    sparsek_jvp,
    sparsek_partial,
    sparsek_st,
    stream_mask,
    topk_hard,
)
from . import ops  # noqa: F401

__all__ = [
    "ArgumentError", "ConfigError", "DecodeSession", "NumericError", "ShapeError", "IoError", "Stream",
    "PartialSortStats", "SelectionMask", "__version__", "attention", "attention_backward", "attention_grads",
    "attention_with_tape", "chunked_forward", "dense_attention", "dense_attention_grads", "linear_mix_attention",
    "linear_mix_attention_grads", "sparsek",
    "sparsek_jvp", "sparsek_partial", "sparsek_st", "stream_mask", "topk_hard", "ops",
]
