"""Device-resident incremental SparseK stream: the reference's ``Stream``
(StreamState, proj/include/sparsek/stream.hpp:26-72; pybind surface
proj/bindings/module.cpp:101-128) over skb_stream_* (include/sparsek_b200.h).

Each ``push`` is one kernel and one device round trip (skb_stream_push_step
returns tau, t, inserted and the survivors popped by that push);
``solution``/``mask`` are computed on the device (skb_stream_solution).
Batches of scores go through ``push_many`` (one launch for n pushes)."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from ._lib import ArgumentError, NumericError, check


def _st():
    return torch.cuda.current_stream().cuda_stream


class SelectionMask:
    """SelectionMask (proj/include/sparsek/selection.hpp:43-49) over the survivors
    of a stream (stream_mask, proj/src/stream.cpp:199-222): ``hard`` = the
    top-floor(k) indicator, ``soft`` = the SparseK weights, ``indices`` = the
    positions of the hard set (ascending); hard/soft follow ``positions``."""

    def __init__(self, positions, hard, soft):
        self.positions = positions
        self.hard = hard
        self.soft = soft
        self.indices = positions[hard == 1.0]
        self.mode = "soft"


class Stream:
    """Push scores one at a time and read the same solution the batch solver
    gives on the prefix. Evictions are permanent; tau never decreases."""

    def __init__(self, k, heap_cap=0, capacity=1 << 16):
        k = float(k)
        if not (k > 0.0) or not math.isfinite(k):
            raise ArgumentError("KBudget: k must be positive and finite")
        self._k = k
        self._cap = int(capacity)
        self._h = C.c_void_p()
        check(_lib.load().skb_stream_create(k, int(heap_cap), self._cap, C.byref(self._h)))
        self._init_common()

    def _init_common(self):
        self._dev = torch.device("cuda", torch.cuda.current_device())
        # room for every index one push can evict (at most the capacity)
        self._ev = (C.c_int64 * self._cap)()
        self._step = _lib.StreamStep()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().skb_stream_destroy(h)
            except Exception:
                pass

    def serialize(self) -> bytes:
        """The reference's wire format (StreamState::serialize,
        proj/src/stream.cpp:224-252): readable by StreamState::deserialize."""
        n = C.c_size_t()
        lib = _lib.load()
        check(lib.skb_stream_serialize(self._h, None, C.byref(n), _st()))
        buf = (C.c_uint8 * n.value)()
        check(lib.skb_stream_serialize(self._h, buf, C.byref(n), _st()))
        return bytes(buf)[: n.value]

    @classmethod
    def deserialize(cls, blob: bytes, capacity=1 << 16):
        """A stream from a blob of the reference's format (either origin)."""
        self = cls.__new__(cls)
        self._cap = int(capacity)
        self._h = C.c_void_p()
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(_lib.load().skb_stream_deserialize(buf, len(blob), self._cap, C.byref(self._h)))
        self._init_common()
        self._k = self._info().k
        return self

    def _info(self):
        info = _lib.StreamInfo()
        check(_lib.load().skb_stream_query(self._h, C.byref(info), _st()))
        return info

    def push(self, z):
        """StreamState::push (proj/src/stream.cpp:72-152) -> {tau, t, inserted,
        evicted}; ``evicted`` lists the survivors this push removed."""
        z = float(z)
        if not math.isfinite(z):
            raise NumericError("stream_push: non-finite value")
        st = self._step
        check(_lib.load().skb_stream_push_step(self._h, z, C.byref(st), self._ev, len(self._ev), _st()))
        evicted = self._ev[: int(st.n_evicted)]
        tau = float(st.tau)
        return {"tau": tau if math.isfinite(tau) else None, "t": int(st.t),
                "inserted": bool(st.inserted), "evicted": evicted}

    def push_many(self, z):
        """Push a batch of scores in one launch; returns (tau, inserted) per push."""
        zt = torch.as_tensor(np.asarray(z, np.float64), device=self._dev).contiguous()
        if not torch.isfinite(zt).all():
            raise NumericError("stream_push: non-finite value")
        n = zt.numel()
        tau = torch.empty(n, dtype=torch.float64, device=self._dev)
        ins = torch.empty(n, dtype=torch.uint8, device=self._dev)
        check(_lib.load().skb_stream_push(self._h, zt.data_ptr(), n, tau.data_ptr(), ins.data_ptr(), _st()))
        return tau, ins.bool()

    def _solution_dev(self, want_hard):
        n = max(1, self.survivors)
        p = torch.empty(n, dtype=torch.float64, device=self._dev)
        idx = torch.empty(n, dtype=torch.int64, device=self._dev)
        hard = torch.empty(n, dtype=torch.uint8, device=self._dev) if want_hard else None
        info = _lib.StreamSolutionInfo()
        check(_lib.load().skb_stream_solution(self._h, p.data_ptr(), idx.data_ptr(),
                                              hard.data_ptr() if want_hard else None, C.byref(info), _st()))
        m = int(info.n)
        return p[:m], idx[:m], (hard[:m] if want_hard else None), info

    def solution(self):
        """{p, tau, u_count, w_count, degenerate} over the full prefix
        (StreamState::solution, proj/src/stream.cpp:154-192); p is computed on
        the device and scattered to the prefix length."""
        p, idx, _, info = self._solution_dev(False)
        full = torch.zeros(int(info.t), dtype=torch.float64, device=self._dev)
        if idx.numel():
            full[idx] = p
        tau = float(info.tau)
        return {"p": full.cpu().numpy(), "tau": tau if math.isfinite(tau) else None,
                "u_count": int(info.u_count), "w_count": int(info.w_count),
                "degenerate": bool(info.degenerate)}

    def mask(self) -> SelectionMask:
        """stream_mask (proj/src/stream.cpp:199-222); ArgumentError on an empty state."""
        if self.t == 0:
            raise ArgumentError("stream_mask: empty state")
        p, idx, hard, _ = self._solution_dev(True)
        return SelectionMask(idx.cpu().numpy(), hard.double().cpu().numpy(), p.cpu().numpy())

    @property
    def tau(self):
        t = self._info().tau
        return t if math.isfinite(t) else None

    @property
    def t(self):
        return int(self._info().t)

    @property
    def survivors(self):
        return int(self._info().survivors)

    def is_evicted(self, index):
        info = self._info()
        index = int(index)
        if not (0 <= index < info.t):
            raise IndexError("is_evicted: index out of range")
        ev = np.zeros(max(info.t, 1), np.uint8)
        check(_lib.load().skb_stream_survivors(self._h, None, None, ev.ctypes.data, _st()))
        return bool(ev[index])


def stream_mask(stream: Stream) -> SelectionMask:
    return stream.mask()
