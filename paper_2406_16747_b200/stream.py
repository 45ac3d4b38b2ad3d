"""Device-resident incremental SparseK stream: the reference's ``Stream``
(StreamState, proj/include/sparsek/stream.hpp:26-72; pybind surface
proj/bindings/module.cpp:101-128) over skb_stream_* (include/sparsek_b200.h)."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from ._lib import ArgumentError, NumericError, check


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
        self._dev = torch.device("cuda", torch.cuda.current_device())
        self._tau = torch.empty(1, dtype=torch.float64, device=self._dev)
        self._ins = torch.empty(1, dtype=torch.uint8, device=self._dev)

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
        st = torch.cuda.current_stream().cuda_stream
        check(lib.skb_stream_serialize(self._h, None, C.byref(n), st))
        buf = (C.c_uint8 * n.value)()
        check(lib.skb_stream_serialize(self._h, buf, C.byref(n), st))
        return bytes(buf)[: n.value]

    @classmethod
    def deserialize(cls, blob: bytes, capacity=1 << 16):
        """A stream from a blob of the reference's format (either origin)."""
        self = cls.__new__(cls)
        self._cap = int(capacity)
        self._h = C.c_void_p()
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(_lib.load().skb_stream_deserialize(buf, len(blob), self._cap, C.byref(self._h)))
        self._k = self._info().k
        self._dev = torch.device("cuda", torch.cuda.current_device())
        self._tau = torch.empty(1, dtype=torch.float64, device=self._dev)
        self._ins = torch.empty(1, dtype=torch.uint8, device=self._dev)
        return self

    def _info(self):
        info = _lib.StreamInfo()
        check(_lib.load().skb_stream_query(self._h, C.byref(info),
                                            torch.cuda.current_stream().cuda_stream))
        return info

    def push(self, z):
        z = float(z)
        if not math.isfinite(z):
            raise NumericError("stream_push: non-finite value")
        zt = torch.tensor([z], dtype=torch.float64, device=self._dev)
        before = self._info()
        check(_lib.load().skb_stream_push(self._h, zt.data_ptr(), 1, self._tau.data_ptr(),
                                           self._ins.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
        tau = float(self._tau.item())
        inserted = bool(self._ins.item())
        _, _, ev = self._survivors()
        prev = getattr(self, "_ev_prev", np.zeros(0, bool))
        new = ev.copy()
        new[: len(prev)] &= ~prev
        if not inserted:  # a rejected arrival is flagged but not reported (stream.cpp:83-88)
            new[before.t] = False
        self._ev_prev = ev
        return {"tau": tau if math.isfinite(tau) else None, "t": before.t + 1,
                "inserted": inserted, "evicted": [int(i) for i in np.nonzero(new)[0]]}

    def _survivors(self):
        info = self._info()
        vals = np.zeros(max(info.survivors, 1))
        idx = np.zeros(max(info.survivors, 1), np.int64)
        ev = np.zeros(max(info.t, 1), np.uint8)
        check(_lib.load().skb_stream_survivors(
            self._h, vals.ctypes.data, idx.ctypes.data, ev.ctypes.data,
            torch.cuda.current_stream().cuda_stream))
        return vals[: info.survivors], idx[: info.survivors], ev[: info.t].astype(bool)

    def solution(self):
        """{p, tau, u_count, w_count, degenerate} over the full prefix
        (StreamState::solution, proj/src/stream.cpp:154-192)."""
        info = self._info()
        vals, idx, _ = self._survivors()
        p = np.zeros(info.t)
        if info.t < self._k:
            p[idx] = 1.0
            return {"p": p, "tau": None, "u_count": len(idx), "w_count": len(idx),
                    "degenerate": True}
        pv = np.clip(vals - info.tau, 0.0, 1.0)
        p[idx] = pv
        uc = int(np.sum(pv == 1.0))
        wc = int(np.sum(pv > 0.0))
        return {"p": p, "tau": info.tau, "u_count": uc, "w_count": wc,
                "degenerate": bool(wc == uc)}

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
        _, _, ev = self._survivors()
        return bool(ev[int(index)])
