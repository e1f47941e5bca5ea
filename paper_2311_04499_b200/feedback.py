"""Python host mirror of the reference's baseline compressors and generic
error-feedback wrapper over the B200 C-ABI.

=========================  =====================================================
this module                reference (paths relative to /root/reference/proj)
=========================  =====================================================
IdentityFilter             compress.hpp:106-110, compress.cpp:246-248
CovapFilter                compress.hpp:112-120, compress.cpp:250-264
TopkFilter                 compress.hpp:122-130, compress.cpp:266-281
RandomkFilter              compress.hpp:132-141, compress.cpp:283-298
Fp16Filter                 compress.hpp:143-147, compress.cpp:300-309
ErrorFeedback              compress.hpp:151-164, compress.cpp:316-344
ErrorFeedback.sync         the non-COVAP branch of train(), trainer.cpp:387-403
topk_compress              compress.hpp:75-76, compress.cpp:119-133
randomk_compress           compress.hpp:78-81, compress.cpp:135-143
fp16_roundtrip             compress.hpp:83-85, compress.cpp:226-236
sparsifier_k               compress.cpp:107-116
=========================  =====================================================

Tensors are flat CUDA tensors (tensors laid out back to back, as
split_by_tensors builds them, trainer.cpp:238-246); every call launches the
sm_100a kernels of libcovap_b200.so (covap_feedback.cu) on the current torch
stream.  Nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _lib as L
from .covap import (EfSchedule, SelectionRule, _CudaArray, _dtype_code, _ptr, _stream_ptr,
                    _torch, require_device)
from .errors import InvalidInput, InvalidState

IDENTITY, COVAP, TOPK, RANDOMK, FP16 = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class IdentityFilter:
    kind = IDENTITY

    def c(self):
        return L.FilterC(IDENTITY, 1, 0, 0.0, 0)


@dataclass(frozen=True)
class CovapFilter:
    interval: int
    rule: int = SelectionRule.kMatchStep
    kind = COVAP

    def c(self):
        return L.FilterC(COVAP, int(self.interval), int(self.rule), 0.0, 0)


@dataclass(frozen=True)
class TopkFilter:
    k_fraction: float
    kind = TOPK

    def c(self):
        return L.FilterC(TOPK, 1, 0, float(self.k_fraction), 0)


@dataclass(frozen=True)
class RandomkFilter:
    k_fraction: float
    seed: int
    kind = RANDOMK

    def c(self):
        return L.FilterC(RANDOMK, 1, 0, float(self.k_fraction), int(self.seed) & (2**64 - 1))


@dataclass(frozen=True)
class Fp16Filter:
    kind = FP16

    def c(self):
        return L.FilterC(FP16, 1, 0, 0.0, 0)


def sparsifier_k(d: int, k_fraction: float) -> int:
    k = ctypes.c_uint64()
    L.lib().covap_sparsifier_k(int(d), float(k_fraction), ctypes.byref(k))
    return k.value


class ErrorFeedback:
    """ErrorFeedback (compress.hpp:151-164) around one filter, resident on one
    GPU: the residual arena and the filter's scratch (histograms, candidate
    lists, wire buffers)."""

    def __init__(self, numels: Sequence[int], schedule: Optional[EfSchedule] = None,
                 filter=None, dtype=None, device: int = 0):
        torch = _torch()
        require_device()
        if filter is None:
            raise InvalidInput("a filter is required")
        self.numels = [int(n) for n in numels]
        self.total = sum(self.numels)
        self.filter = filter
        self.schedule = schedule if schedule is not None else EfSchedule()
        self.dtype = torch.float32 if dtype is None else dtype
        self.dtype_code = _dtype_code(self.dtype)
        self.device = int(device)
        arr = (ctypes.c_uint64 * max(len(self.numels), 1))(*self.numels)
        efc, fc = self.schedule.c(), filter.c()
        h = ctypes.c_void_p()
        L.lib().covap_feedback_create(arr, len(self.numels), self.dtype_code, ctypes.byref(efc),
                                      ctypes.byref(fc), self.device, ctypes.byref(h))
        self._h = h
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        L.lib().covap_feedback_residual(h, ctypes.byref(p), ctypes.byref(n))
        self.residuals = torch.as_tensor(_CudaArray(p.value, n.value, self.dtype_code),
                                         device=torch.device("cuda", self.device))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._LIB is not None:
            L._LIB.covap_feedback_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def num_steps(self) -> int:
        v = ctypes.c_uint64()
        L.lib().covap_feedback_get_step(self._h, ctypes.byref(v))
        return v.value

    @num_steps.setter
    def num_steps(self, v: int):
        L.lib().covap_feedback_set_step(self._h, int(v))

    def reset(self, stream=None):
        L.lib().covap_feedback_reset(self._h, _stream_ptr(stream, self.device))

    def _check(self, t):
        if t.dtype != self.dtype or not t.is_cuda or not t.is_contiguous():
            raise InvalidInput("tensor must be a contiguous CUDA tensor of the state's dtype")
        if t.numel() != self.total:
            raise InvalidState("gradient tensor count does not match error-feedback state")

    def step(self, gradients, kept=None, stream=None):
        """ErrorFeedback::step (compress.cpp:323-344): returns the kept
        (filtered, compensated) gradient; residuals and num_steps advance."""
        self._check(gradients)
        if kept is None:
            kept = _torch().empty_like(gradients)
        self._check(kept)
        L.lib().covap_feedback_step(self._h, _ptr(gradients), _ptr(kept),
                                    _stream_ptr(stream, self.device))
        return kept

    def transmitted_elements(self, step: Optional[int] = None) -> int:
        """GradientFilter::transmitted_elements (compress.cpp:246-314)."""
        e = ctypes.c_uint64()
        L.lib().covap_feedback_transmitted(self._h, self.num_steps if step is None else int(step),
                                           ctypes.byref(e), None)
        return e.value

    def wire_bytes(self, step: Optional[int] = None) -> int:
        """Bytes train() accounts for one step (trainer.cpp:396-400)."""
        b = ctypes.c_uint64()
        L.lib().covap_feedback_transmitted(self._h, self.num_steps if step is None else int(step),
                                           None, ctypes.byref(b))
        return b.value

    def saturations(self, stream=None) -> int:
        v = ctypes.c_uint64()
        L.lib().covap_feedback_saturations(self._h, ctypes.byref(v),
                                           _stream_ptr(stream, self.device))
        return v.value

    # -- synchronisation (trainer.cpp:387-403) ----------------------------
    def sync(self, grad, out, comm=None, stream=None):
        """Error-feedback step + exchange + rank-ordered mean of every rank's
        kept gradient into out."""
        self._check(grad)
        self._check(out)
        L.lib().covap_feedback_sync_step(self._h, comm.handle if comm is not None else None,
                                         _ptr(grad), _ptr(out), _stream_ptr(stream, self.device))

    def pack(self, grad, out, stream=None):
        self._check(grad)
        self._check(out)
        L.lib().covap_feedback_pack(self._h, _ptr(grad), _ptr(out),
                                    _stream_ptr(stream, self.device))

    def wire(self):
        """(a, b) torch views of this rank's wire payload (uint8), None when
        unused: fp16 halves / top-k indices, values."""
        torch = _torch()
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        ba, bb = ctypes.c_uint64(), ctypes.c_uint64()
        L.lib().covap_feedback_wire(self._h, ctypes.byref(a), ctypes.byref(ba), ctypes.byref(b),
                                    ctypes.byref(bb))
        dev = torch.device("cuda", self.device)

        def view(p, n):
            if not p.value or not n.value:
                return None
            arr = _CudaArray(p.value, n.value, L.F32)
            arr.__cuda_array_interface__["typestr"] = "|u1"
            return torch.as_tensor(arr, device=dev)
        return view(a, ba), view(b, bb)

    def combine(self, recv_a, recv_b, P: int, out, stream=None):
        self._check(out)
        L.lib().covap_feedback_combine(self._h, None if recv_a is None else _ptr(recv_a),
                                       None if recv_b is None else _ptr(recv_b), int(P), _ptr(out),
                                       _stream_ptr(stream, self.device))


def _device_of(x):
    return x.device.index if x.device.index is not None else 0


def topk_compress(x, k_fraction: float, stream=None):
    """topk_compress (compress.cpp:119-133): (indices int64, values) on the
    device, largest magnitude first, ties to the lower index."""
    torch = _torch()
    dev = _device_of(x)
    idx = torch.empty(max(x.numel(), 1), dtype=torch.int64, device=x.device)
    val = torch.empty(max(x.numel(), 1), dtype=x.dtype, device=x.device)
    k = ctypes.c_uint64()
    L.lib().covap_topk_compress(dev, _dtype_code(x.dtype), _ptr(x), x.numel(), float(k_fraction),
                                _ptr(idx), _ptr(val), ctypes.byref(k), _stream_ptr(stream, dev))
    return idx[:k.value], val[:k.value]


def randomk_compress(x, k_fraction: float, seed: int, stream=None):
    """randomk_compress (compress.cpp:135-143): ascending indices sampled
    without replacement from SplitMix64(seed), and their values."""
    torch = _torch()
    dev = _device_of(x)
    idx = torch.empty(max(x.numel(), 1), dtype=torch.int64, device=x.device)
    val = torch.empty(max(x.numel(), 1), dtype=x.dtype, device=x.device)
    k = ctypes.c_uint64()
    L.lib().covap_randomk_compress(dev, _dtype_code(x.dtype), _ptr(x), x.numel(), float(k_fraction),
                                   int(seed) & (2**64 - 1), _ptr(idx), _ptr(val), ctypes.byref(k),
                                   _stream_ptr(stream, dev))
    return idx[:k.value], val[:k.value]


def fp16_roundtrip(x, stream=None):
    """fp16_roundtrip (compress.cpp:226-236): (widened values, saturation count)."""
    torch = _torch()
    dev = _device_of(x)
    out = torch.empty_like(x)
    sat = ctypes.c_uint64()
    L.lib().covap_fp16_roundtrip(dev, _dtype_code(x.dtype), _ptr(x), x.numel(), _ptr(out),
                                 ctypes.byref(sat), _stream_ptr(stream, dev))
    return out, sat.value
