"""Python host mirror of the reference COVAP API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(paths relative to /root/reference/proj):

=========================  =====================================================
this module                reference
=========================  =====================================================
LayerSpec / ModelSpec      model.hpp:13-31
allocate_buckets           model.hpp:82-83, model.cpp:36-60
median_numel               model.hpp:87, model.cpp:66-82
shard_plan                 model.hpp:89-92, model.cpp:95-115
effective_tensors/_numels  model.hpp:94-95, model.cpp:117-143
SelectionRule              compress.hpp:15-19
select_tensors             compress.hpp:22-24, compress.cpp:13-28
EfSchedule/ef_coefficient  compress.hpp:26-34, compress.cpp:30-35
CovapConfig                compress.hpp:36-40
CompressorState.zeros      compress.hpp:42-47, compress.cpp:37-42 (device arena)
covap_compress             compress.hpp:57-61, compress.cpp:50-85  (kernel K1)
covap_decompress           compress.hpp:63-65, compress.cpp:87-103 (kernel K2)
allreduce_mean             trainer.hpp:56-58, trainer.cpp:35-47    (NCCL + K2)
ccr / choose_interval      perf.hpp:24-28, perf.cpp:40-53
profile_ccr                sim.hpp:84-96, sim.cpp:164-216
=========================  =====================================================

Data lives on the GPU as flat torch tensors laid out bucket by bucket (the
layout train() builds with split_by_tensors, trainer.cpp:238-246); every
compute call launches the sm_100a kernels of libcovap_b200.so on the current
torch stream.  Nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _lib as L
from .errors import InvalidInput, InvalidState, NoDeviceError  # noqa: F401

_LAYOUT_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "layouts")
DEFAULT_BUCKET_CAP_BYTES = 25 * 1024 * 1024  # model.hpp:26


class SelectionRule:
    """compress.hpp:15-19: kMatchStep keeps t at step s iff t == s (mod K)."""
    kMatchStep = 0
    kPlusStep = 1


@dataclass
class LayerSpec:
    name: str
    param_count: int
    bytes_per_param: int = 4
    backward_ms: float = 0.0

    def bytes(self) -> int:
        return self.param_count * self.bytes_per_param


@dataclass
class ModelSpec:
    layers: List[LayerSpec] = field(default_factory=list)
    bucket_cap_bytes: int = DEFAULT_BUCKET_CAP_BYTES
    name: str = ""

    def total_params(self) -> int:
        return sum(l.param_count for l in self.layers)

    @staticmethod
    def from_json(doc) -> "ModelSpec":
        """model_from_json (model.cpp:170-186)."""
        if isinstance(doc, str):
            doc = json.loads(doc)
        if not isinstance(doc, dict) or not isinstance(doc.get("layers"), list):
            raise InvalidInput("model JSON must be an object with a 'layers' array")
        layers = []
        for i, lj in enumerate(doc["layers"]):
            name = lj.get("name", f"layer{i}")
            if "param_count" not in lj:
                raise InvalidInput(f"layer '{name}' missing param_count")
            layers.append(LayerSpec(name, int(lj["param_count"]), int(lj.get("bytes_per_param", 4)),
                                    float(lj.get("backward_ms", 0.0))))
        return ModelSpec(layers, int(doc.get("bucket_cap_bytes", DEFAULT_BUCKET_CAP_BYTES)),
                         doc.get("name", ""))


def load_layout(name: str) -> ModelSpec:
    """Gradient layouts of BASELINE.json's configs:
    resnet50, vgg16, bert_large, tablev."""
    with open(os.path.join(_LAYOUT_DIR, name + ".json")) as f:
        return ModelSpec.from_json(json.load(f))


@dataclass
class EfSchedule:
    enabled: bool = True
    init_value: float = 0.3
    ascend_steps: int = 100
    ascend_range: float = 0.1

    def c(self):
        return L.EfC(1 if self.enabled else 0, float(self.init_value), int(self.ascend_steps),
                     float(self.ascend_range))


@dataclass
class CovapConfig:
    interval: int = 1
    rule: int = SelectionRule.kMatchStep
    ef: EfSchedule = field(default_factory=EfSchedule)


@dataclass(frozen=True)
class Bucket:
    index: int
    numel: int
    begin: int
    layer_refs: tuple


@dataclass(frozen=True)
class EffectiveTensor:
    bucket: int
    begin: int
    end: int

    def numel(self) -> int:
        return self.end - self.begin


def _u64(seq):
    return (ctypes.c_uint64 * max(len(seq), 1))(*[int(x) for x in seq])


class BucketPlan:
    """A native covap_plan handle: buckets, effective tensors and the
    per-phase send layout.  ``interval``/``rule`` fix the selection phases."""

    def __init__(self, model: ModelSpec, cap_bytes: Optional[int] = None, interval: int = 1,
                 rule: int = SelectionRule.kMatchStep, shard: int = -1, pad: bool = False):
        lib = L.lib()
        self.model = model
        self.cap_bytes = int(model.bucket_cap_bytes if cap_bytes is None else cap_bytes)
        numel = _u64([l.param_count for l in model.layers])
        bpp = (ctypes.c_uint32 * max(len(model.layers), 1))(*[l.bytes_per_param for l in model.layers])
        h = ctypes.c_void_p()
        if int(interval) < 1:
            raise InvalidInput("shard interval must be >= 1")
        lib.covap_plan_create_ex(numel, bpp, len(model.layers), self.cap_bytes, int(interval),
                                 int(rule), int(shard), 1 if pad else 0, ctypes.byref(h))
        self._h = h
        info = L.PlanInfoC()
        lib.covap_plan_get_info(h, ctypes.byref(info))
        self.info = info
        nb, nt = info.n_buckets, info.n_tensors
        bn, bb, bf, bl = (ctypes.c_uint64 * nb)(), (ctypes.c_uint64 * nb)(), (ctypes.c_uint64 * nb)(), (ctypes.c_uint64 * nb)()
        lib.covap_plan_buckets(h, bn, bb, bf, bl)
        self.buckets = [Bucket(i, bn[i], bb[i], tuple(range(bf[i], bf[i] + bl[i]))) for i in range(nb)]
        tb, tbeg, tend = (ctypes.c_uint64 * nt)(), (ctypes.c_uint64 * nt)(), (ctypes.c_uint64 * nt)()
        lib.covap_plan_tensors(h, tb, tbeg, tend)
        self.tensors = [EffectiveTensor(tb[i], tbeg[i], tend[i]) for i in range(nt)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._LIB is not None:
            L._LIB.covap_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def interval(self) -> int:
        return self.info.interval

    @property
    def rule(self) -> int:
        return self.info.rule

    @property
    def sharded(self) -> bool:
        return bool(self.info.sharded)

    @property
    def twice_median(self) -> int:
        return self.info.twice_median

    @property
    def max_send_elems(self) -> int:
        return self.info.max_send_elems

    def total_numel(self) -> int:
        return self.info.total_numel

    def device_numel(self) -> int:
        """Length of device-side arenas: N, plus bucket padding for a padded plan."""
        return self.info.device_numel

    @property
    def padded(self) -> bool:
        return bool(self.info.padded)

    def device_begin(self, bucket: int) -> int:
        return self.bucket_range(0, bucket).device_begin

    def selection(self, step: int) -> List[int]:
        keep = (ctypes.c_uint8 * len(self.tensors))()
        L.lib().covap_plan_selection(self._h, int(step), keep)
        return [t for t in range(len(self.tensors)) if keep[t]]

    def bucket_range(self, step: int, bucket: int) -> L.BucketRangeC:
        r = L.BucketRangeC()
        L.lib().covap_plan_bucket_range(self._h, int(step), int(bucket), ctypes.byref(r))
        return r

    def send_elems(self, step: int):
        s, p = ctypes.c_uint64(), ctypes.c_uint64()
        L.lib().covap_plan_send_elems(self._h, int(step), ctypes.byref(s), ctypes.byref(p))
        return s.value, p.value

    def payload_elements(self, step: int) -> int:
        return self.send_elems(step)[1]


# ------------------------------------------------------------------ planner

def allocate_buckets(model: ModelSpec, cap_bytes: Optional[int] = None) -> BucketPlan:
    """Greedy bucketing, no sharding (model.cpp:36-60)."""
    return BucketPlan(model, cap_bytes, interval=1, shard=0)


def median_numel(plan: BucketPlan) -> float:
    """MedianNumel::value() (model.hpp:55) of the plan's buckets."""
    return plan.twice_median / 2.0


def shard_plan(plan: BucketPlan, interval: int, rule: int = SelectionRule.kMatchStep) -> BucketPlan:
    """shard_plan (model.cpp:95-115); the result carries `interval` phases."""
    return BucketPlan(plan.model, plan.cap_bytes, interval=interval, rule=rule, shard=1)


def plan_for(model: ModelSpec, config: CovapConfig, pad: bool = False) -> BucketPlan:
    """The plan train() builds: allocate, then shard only when K > 1
    (trainer.cpp:266-271).  pad=True: the padded device layout the
    bucket-local (DDP GradBucket) calls need."""
    return BucketPlan(model, None, interval=config.interval, rule=config.rule, shard=-1, pad=pad)


def effective_tensors(plan: BucketPlan) -> List[EffectiveTensor]:
    return list(plan.tensors)


def effective_numels(plan: BucketPlan) -> List[int]:
    return [t.numel() for t in plan.tensors]


# --------------------------------------------------------- scalar helpers

def select_tensors(num_steps: int, interval: int, tensor_count: int,
                   rule: int = SelectionRule.kMatchStep) -> List[int]:
    if tensor_count < 1 or interval < 1:
        keep = (ctypes.c_uint8 * 1)()
    else:
        keep = (ctypes.c_uint8 * tensor_count)()
    L.lib().covap_select_tensors(int(num_steps), int(interval), int(tensor_count), int(rule), keep)
    return [t for t in range(tensor_count) if keep[t]]


def ef_coefficient(num_steps: int, schedule: EfSchedule) -> float:
    out = ctypes.c_double()
    ef = schedule.c()
    L.lib().covap_ef_coefficient(int(num_steps), ctypes.byref(ef), ctypes.byref(out))
    return out.value


def ccr(comm_ms: float, comp_ms: float) -> float:
    out = ctypes.c_double()
    L.lib().covap_ccr(float(comm_ms), float(comp_ms), ctypes.byref(out))
    return out.value


def choose_interval(ccr_value: float) -> int:
    out = ctypes.c_uint32()
    L.lib().covap_choose_interval(float(ccr_value), ctypes.byref(out))
    return out.value


@dataclass
class ProfileResult:
    ccr: float
    comp_ms: float
    comm_aligned_ms: float
    naive_comm_ms: List[float]
    recommended_interval: int


def profile_ccr(comm_start: Sequence[Sequence[float]], comm_end: Sequence[float],
                comp_ms: float, expected_workers: int) -> ProfileResult:
    """profile_ccr (sim.cpp:164-216) over gathered per-worker arrivals."""
    W = len(comm_start)
    C = len(comm_end)
    starts = (ctypes.c_double * max(W * C, 1))(*[float(x) for row in comm_start for x in row])
    ends = (ctypes.c_double * max(C, 1))(*[float(x) for x in comm_end])
    naive = (ctypes.c_double * max(W, 1))()
    aligned, c, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    L.lib().covap_profile_ccr(starts, ends, W, int(expected_workers), C, float(comp_ms),
                              ctypes.byref(aligned), naive, ctypes.byref(c), ctypes.byref(k))
    return ProfileResult(c.value, float(comp_ms), aligned.value, list(naive[:W]), k.value)


# ------------------------------------------------------------ device side

def _torch():
    import torch
    return torch


def _dtype_code(dtype) -> int:
    torch = _torch()
    if dtype == torch.float32:
        return L.F32
    if dtype == torch.float64:
        return L.F64
    raise InvalidInput("dtype must be torch.float32 or torch.float64")


class _CudaArray:
    """Zero-copy view of a device allocation owned by the native library."""

    def __init__(self, ptr, n, dtype_code):
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": "<f8" if dtype_code == L.F64 else "<f4",
            "data": (int(ptr), False), "version": 3, "strides": None}


def _stream_ptr(stream=None, device=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def require_device():
    n = ctypes.c_int()
    L.lib().covap_device_count(ctypes.byref(n))  # raises NoDeviceError without a GPU
    return n.value


class CompressorState:
    """CompressorState (compress.hpp:42-47) resident on one GPU: the flat
    residual arena (offsets = flat gradient offsets), num_steps, the send
    scratch and the comm side stream."""

    def __init__(self, plan: BucketPlan, dtype=None, device: int = 0,
                 ef: Optional[EfSchedule] = None):
        torch = _torch()
        require_device()
        self.plan = plan
        self.dtype = torch.float32 if dtype is None else dtype
        self.dtype_code = _dtype_code(self.dtype)
        self.device = int(device)
        self.ef = ef if ef is not None else EfSchedule()
        efc = self.ef.c()
        h = ctypes.c_void_p()
        L.lib().covap_state_create(plan.handle, self.dtype_code, self.device, ctypes.byref(efc),
                                   ctypes.byref(h))
        self._h = h
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        L.lib().covap_state_residual(h, ctypes.byref(p), ctypes.byref(n))
        dev = torch.device("cuda", self.device)
        self.residuals = torch.as_tensor(_CudaArray(p.value, n.value, self.dtype_code), device=dev)
        L.lib().covap_state_send(h, ctypes.byref(p), ctypes.byref(n))
        self.send = torch.as_tensor(_CudaArray(p.value, n.value, self.dtype_code), device=dev)

    @staticmethod
    def zeros(plan: BucketPlan, dtype=None, device: int = 0, ef=None) -> "CompressorState":
        return CompressorState(plan, dtype, device, ef)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._LIB is not None:
            L._LIB.covap_state_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def num_steps(self) -> int:
        v = ctypes.c_uint64()
        L.lib().covap_state_get_step(self._h, ctypes.byref(v))
        return v.value

    @num_steps.setter
    def num_steps(self, v: int):
        L.lib().covap_state_set_step(self._h, int(v))

    def set_fused(self, fuse_single_rank: bool):
        """One rank: fused K1F pass (default) or the multi-rank K1 -> C1 -> K2 path."""
        L.lib().covap_state_set_fused(self._h, 1 if fuse_single_rank else 0)

    def set_free_sms(self, n: int):
        """The overlapped multi-rank schedules run K1 / K2 on all SMs but n,
        which stay free for the allreduce kernels beside them."""
        L.lib().covap_state_set_free_sms(self._h, int(n))

    def set_pipeline(self, groups: int):
        """Multi-rank sync step as `groups` bucket groups whose allreduces
        overlap the later groups' K1 (1 = serial)."""
        L.lib().covap_state_set_pipeline(self._h, int(groups))

    def use_symmetric(self, comm: "Communicator"):
        """Send buffer -> an NCCL symmetric window on ``comm`` (collective;
        NVLS / symmetric-memory allreduce kernels at P > 1)."""
        L.lib().covap_state_use_symmetric(self._h, comm.handle)
        torch = _torch()
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        L.lib().covap_state_send(self._h, ctypes.byref(p), ctypes.byref(n))
        self.send = torch.as_tensor(_CudaArray(p.value, n.value, self.dtype_code),
                                    device=torch.device("cuda", self.device))

    def set_host_ramp(self, ramp_min_elems: int):
        """Smallest chunk of sync_host's geometric ramp at both ends of the step."""
        L.lib().covap_state_set_host_ramp(self._h, int(ramp_min_elems))

    def reset(self, stream=None):
        L.lib().covap_state_reset(self._h, _stream_ptr(stream, self.device))

    # -- kernels ---------------------------------------------------------
    def filter_pack(self, grad, b0: int = 0, b1: Optional[int] = None, send=None, stream=None,
                    out=None):
        """K1 over buckets [b0, b1) at the current step.  With ``out``, K1 also
        zero-fills the unselected output (the multi-rank step's split; pair
        it with ``unpack(..., selected_only=True)``)."""
        self._check(grad)
        b1 = len(self.plan.buckets) if b1 is None else b1
        snd = None if send is None else _ptr(send)
        if out is None:
            L.lib().covap_filter_pack(self._h, _ptr(grad), snd, int(b0), int(b1),
                                      _stream_ptr(stream, self.device))
        else:
            self._check(out)
            L.lib().covap_filter_pack_zero(self._h, _ptr(grad), snd, _ptr(out), int(b0), int(b1),
                                           _stream_ptr(stream, self.device))

    def unpack(self, out, scale: float = 1.0, mean: bool = True, b0: int = 0,
               b1: Optional[int] = None, recv=None, stream=None, selected_only: bool = False):
        """K2 over buckets [b0, b1) at the current step: selected slots get
        (0 + recv) * scale (mean=True, allreduce_mean's order) or recv * scale
        (mean=False, covap_decompress); the rest is zero-filled — unless
        ``selected_only`` (after a zero-filling K1: only the selected slots
        are written, mean semantics)."""
        self._check(out)
        b1 = len(self.plan.buckets) if b1 is None else b1
        rcv = None if recv is None else _ptr(recv)
        if selected_only:
            L.lib().covap_unpack_selected(self._h, rcv, _ptr(out), float(scale), int(b0), int(b1),
                                          _stream_ptr(stream, self.device))
        else:
            L.lib().covap_unpack(self._h, rcv, _ptr(out), float(scale), 1 if mean else 0,
                                 int(b0), int(b1), _stream_ptr(stream, self.device))

    def filter_unpack(self, grad, out, scale: float = 1.0, b0: int = 0,
                      b1: Optional[int] = None, stream=None):
        """K1F: K1 + K2 fused for a single rank (the allreduce is the identity)."""
        self._check(grad)
        self._check(out)
        b1 = len(self.plan.buckets) if b1 is None else b1
        L.lib().covap_filter_unpack(self._h, _ptr(grad), _ptr(out), float(scale), int(b0), int(b1),
                                    _stream_ptr(stream, self.device))

    def step_end(self):
        L.lib().covap_step_end(self._h)

    def _check(self, t):
        if t.dtype != self.dtype or not t.is_cuda or not t.is_contiguous():
            raise InvalidInput("tensor must be a contiguous CUDA tensor of the state's dtype")
        if t.numel() != self.plan.device_numel():
            raise InvalidState("gradient length does not match the plan")


@dataclass
class CompressedUpdate:
    """CompressedUpdate (compress.hpp:49-55): ``selected`` ascending, the
    payload packed in ``send`` (selected tensors at ``send_offsets``), step."""
    selected: List[int]
    step: int
    send: object
    send_offsets: List[int]
    numels: List[int]
    state: "CompressorState" = None

    def payload_elements(self) -> int:
        return sum(self.numels)

    def payload(self) -> List[object]:
        return [self.send[o:o + n] for o, n in zip(self.send_offsets, self.numels)]


def covap_compress(gradients, state: CompressorState, config: Optional[CovapConfig] = None,
                   stream=None) -> CompressedUpdate:
    """covap_compress (compress.cpp:50-85) on the device: one K1 launch over
    the whole flat gradient, then ++num_steps."""
    plan = state.plan
    if config is not None and (config.interval != plan.interval or config.rule != plan.rule):
        raise InvalidState("config interval/rule differ from the plan the state was built on")
    step = state.num_steps
    state.filter_pack(gradients, stream=stream)
    state.step_end()
    sel = plan.selection(step)
    offs, numels = [], []
    for t in sel:
        ts = plan.tensors[t]
        br = plan.bucket_range(step, ts.bucket)
        offs.append(br.send_offset + (ts.begin - br.sel_begin))
        numels.append(ts.numel())
    return CompressedUpdate(sel, step, state.send, offs, numels, state)


def covap_decompress(update: CompressedUpdate, out=None, recv=None, world: int = 0,
                     stream=None):
    """covap_decompress (compress.cpp:87-103) on the device (K2): payload at
    the selected slots, zeros elsewhere.  With ``world`` = P > 0 the pass also
    applies allreduce_mean's (0 + sum) * 1/P (trainer.cpp:41-45) to a summed
    ``recv`` — the fused unpack/scale of the sync path."""
    state = update.state
    torch = _torch()
    if out is None:
        out = torch.empty(state.plan.device_numel(), dtype=state.dtype,
                          device=torch.device("cuda", state.device))
    saved = state.num_steps
    state.num_steps = update.step
    try:
        if world > 0:
            state.unpack(out, 1.0 / world, True, recv=recv, stream=stream)
        else:
            state.unpack(out, 1.0, False, recv=recv, stream=stream)
    finally:
        state.num_steps = saved
    return out


# ------------------------------------------------------------ communicator

class Communicator:
    """One NCCL rank over NVLink/NVSwitch (C1).  Rendezvous of the unique id
    rides on torch.distributed (plumbing); the data path is NCCL."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        h = ctypes.c_void_p()
        L.lib().covap_comm_create(uid, int(nranks), int(rank), int(device), ctypes.byref(h))
        self._h = h
        self.nranks, self.rank, self.device = int(nranks), int(rank), int(device)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        L.lib().covap_comm_unique_id(buf)
        return buf.raw

    @staticmethod
    def from_torch_distributed(device: int) -> "Communicator":
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Communicator(obj[0], world, rank, device)

    @property
    def handle(self):
        return self._h

    def allreduce(self, buf, stream=None):
        L.lib().covap_allreduce(self._h, _ptr(buf), buf.numel(), _dtype_code(buf.dtype),
                                _stream_ptr(stream, self.device))

    def profile_exchange(self, durations: Sequence[float], comp_ms: float):
        n = len(durations)
        d = (ctypes.c_double * max(n, 1))(*durations)
        a = (ctypes.c_double * max(n, 1))()
        c = ctypes.c_double()
        L.lib().covap_comm_profile_exchange(self._h, d, n, float(comp_ms), a, ctypes.byref(c))
        return list(a[:n]), c.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.lib().covap_comm_destroy(self._h)
            self._h = None


def allreduce_mean(buf, comm: Optional[Communicator] = None, out=None, stream=None):
    """allreduce_mean (trainer.cpp:35-47) of one device buffer per rank: NCCL
    sum in place (P > 1), then out = (0 + sum) * (1/P) — one stream-ordered
    native call (covap_comm_allreduce_mean), no state, no allocation beyond
    ``out``.  fp32 or fp64; ``out`` may be ``buf``."""
    torch = _torch()
    code = _dtype_code(buf.dtype)
    if not buf.is_cuda or not buf.is_contiguous():
        raise InvalidInput("allreduce_mean needs a contiguous CUDA tensor")
    if out is None:
        out = torch.empty_like(buf)
    elif out.dtype != buf.dtype or out.numel() != buf.numel() or not out.is_contiguous():
        raise InvalidInput("allreduce vectors differ in length")  # trainer.cpp:38-39
    L.lib().covap_comm_allreduce_mean(None if comm is None else comm.handle, code, _ptr(buf),
                                      _ptr(out), buf.numel(), _stream_ptr(stream, buf.device))
    return out


# ------------------------------------------------------------ the sync path

class CovapSync:
    """The per-step gradient synchronisation of one rank (trainer.cpp:365-386
    restated for one process per GPU):

    * ``sync(grad, out)`` — standalone: K1 -> NCCL allreduce(sum) of the
      packed selected shards -> K2 (x 1/P, zero fill) -> ++step, on one stream;
    * ``bucket_ready(b, grad, out)`` + ``finish()`` — the overlapped DDP-hook
      schedule: K1(b) on the compute stream, allreduce(b's selected range) and
      K2(b) on the side stream while later buckets are still being produced;
    * ``dense_bucket_ready`` — the no-compression baseline (trainer.cpp:388).
    """

    def __init__(self, plan: BucketPlan, comm: Optional[Communicator] = None, dtype=None,
                 device: int = 0, ef: Optional[EfSchedule] = None,
                 fuse_single_rank: bool = True, pipeline: int = 1, symmetric: bool = False,
                 free_sms: int = 0):
        self.plan = plan
        self.comm = comm
        self.state = CompressorState(plan, dtype, device, ef)
        self.device = device
        if not fuse_single_rank:
            self.state.set_fused(False)
        if pipeline != 1:
            self.state.set_pipeline(pipeline)
        if free_sms:
            self.state.set_free_sms(free_sms)
        if symmetric and comm is not None:
            self.state.use_symmetric(comm)

    @property
    def world(self) -> int:
        return self.comm.nranks if self.comm is not None else 1

    def _c(self):
        return None if self.comm is None else self.comm.handle

    def sync(self, grad, out, stream=None):
        self.state._check(grad)
        self.state._check(out)
        L.lib().covap_sync_step(self.state.handle, self._c(), _ptr(grad), _ptr(out),
                                _stream_ptr(stream, self.device))

    def sync_host(self, host_grad, host_out, dev_grad=None, dev_out=None,
                  chunk_elems: int = 0, stream=None):
        """The sync step on host (pinned) buffers: chunked H2D -> kernels (+
        allreduce) -> D2H on three streams (covap_sync_step_host)."""
        torch = _torch()
        n = self.plan.device_numel()
        if host_grad.numel() != n or host_out.numel() != n:
            raise InvalidState("host buffer length does not match the plan")
        if host_grad.dtype != self.state.dtype or host_out.dtype != self.state.dtype:
            raise InvalidInput("host buffers must have the state's dtype")
        dev = torch.device("cuda", self.device)
        if dev_grad is None:
            if getattr(self, "_stage", None) is None:
                self._stage = torch.empty(n, dtype=self.state.dtype, device=dev)
            dev_grad = self._stage
        dev_out = dev_grad if dev_out is None else dev_out
        L.lib().covap_sync_step_host(self.state.handle, self._c(),
                                     ctypes.c_void_p(host_grad.data_ptr()),
                                     ctypes.c_void_p(host_out.data_ptr()), _ptr(dev_grad),
                                     _ptr(dev_out), int(chunk_elems),
                                     _stream_ptr(stream, self.device))

    def sync_sgd(self, grad, params, lr: float, stream=None):
        """The sync step ending in the SGD update (trainer.cpp:408-409) instead
        of writing a synchronised gradient: params -= lr * update, fused into
        the last kernel (one rank: K1F+SGD; P ranks: K1 -> C1 -> K2+SGD)."""
        self.state._check(grad)
        self.state._check(params)
        L.lib().covap_sync_step_sgd(self.state.handle, self._c(), _ptr(grad), _ptr(params),
                                    float(lr), _stream_ptr(stream, self.device))

    def bucket_ready(self, bucket: int, grad, out, stream=None):
        L.lib().covap_bucket_ready(self.state.handle, self._c(), int(bucket), _ptr(grad), _ptr(out),
                                   _stream_ptr(stream, self.device))

    def bucket_ready_local(self, bucket: int, bucket_grad, bucket_out, stream=None):
        """bucket_ready() with the bucket in its own buffer (a DDP GradBucket);
        needs a padded plan."""
        L.lib().covap_bucket_ready_local(self.state.handle, self._c(), int(bucket), _ptr(bucket_grad),
                                         _ptr(bucket_out), _stream_ptr(stream, self.device))

    def dense_bucket_ready_local(self, bucket: int, bucket_grad, bucket_out, stream=None):
        L.lib().covap_dense_bucket_ready_local(self.state.handle, self._c(), int(bucket),
                                               _ptr(bucket_grad), _ptr(bucket_out),
                                               _stream_ptr(stream, self.device))

    def dense_bucket_ready(self, bucket: int, grad, out, stream=None):
        L.lib().covap_dense_bucket_ready(self.state.handle, self._c(), int(bucket), _ptr(grad),
                                         _ptr(out), _stream_ptr(stream, self.device))

    def finish(self, stream=None):
        L.lib().covap_step_finish(self.state.handle, _stream_ptr(stream, self.device))

    def side_stream(self):
        """The stream bucket_ready() runs each bucket's allreduce and unpack on,
        as a torch ExternalStream."""
        import torch
        p = ctypes.c_void_p()
        L.lib().covap_state_side_stream(self.state.handle, ctypes.byref(p))
        return torch.cuda.ExternalStream(p.value, device=torch.device("cuda", self.device))

    def last_comm_ms(self) -> List[float]:
        n = len(self.plan.buckets)
        d = (ctypes.c_double * n)()
        L.lib().covap_state_last_comm_ms(self.state.handle, d, n)
        return list(d)


# ------------------------------------------------------------ harness

def stream_key(seed: int, rank: int, step: int) -> int:
    return L.lib().covap_stream_key(int(seed), int(rank), int(step))


def generate(out, key: int, kind: int = 0, begin: int = 0, stream=None):
    """K0: fill ``out`` with the synthetic gradient stream ``key``."""
    L.lib().covap_generate(_ptr(out), out.numel(), _dtype_code(out.dtype), int(key), int(kind),
                           int(begin), _stream_ptr(stream, out.device))


def spin(us: float, blocks: int = 1, stream=None, device=None):
    """K3: occupy `blocks` CTAs for `us` microseconds (backward emulator)."""
    L.lib().covap_spin(float(us), int(blocks), _stream_ptr(stream, device))


def busy(us: float, slice_us: float = 50.0, stream=None, device=None):
    """K3, full-GPU form: `us` microseconds of kernels that each own every SM
    (1024 threads + 160 KB shared memory per SM), `slice_us` per kernel."""
    L.lib().covap_busy(float(us), float(slice_us), _stream_ptr(stream, device))


# ------------------------------------------------------------ CCR controller

class NcclExchange:
    """Rank-min of per-collective durations + rank 0's compute time over the
    native NCCL communicator (covap_comm_profile_exchange)."""

    def __init__(self, comm: Optional[Communicator]):
        self.comm = comm

    def __call__(self, durations, comp_ms):
        if self.comm is None:
            return list(durations), float(comp_ms)
        return self.comm.profile_exchange(durations, comp_ms)


class TorchDistExchange:
    """The same exchange over an initialised torch.distributed group (any
    backend; CPU tensors for gloo)."""

    def __call__(self, durations, comp_ms):
        torch = _torch()
        import torch.distributed as dist
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend() == "nccl" else torch.device("cpu")
        d = torch.tensor(list(durations), dtype=torch.float64, device=dev)
        c = torch.tensor([float(comp_ms)], dtype=torch.float64, device=dev)
        if d.numel():
            dist.all_reduce(d, op=dist.ReduceOp.MIN)
        dist.broadcast(c, src=0)
        return d.cpu().tolist(), float(c.item())


@dataclass
class CovapSettings:
    """The "covap" section of an experiment document (config.cpp:133-157):
    ``interval`` (K >= 1) or ``auto_interval`` ("auto": K from the measured
    CCR), the selection rule ("narrative" = kMatchStep, "formula" =
    kPlusStep) and the EF schedule.  Parsed and validated natively
    (covap_settings_from_json): ConfigError carries the field path."""
    interval: int = 1
    auto_interval: bool = False
    rule: int = SelectionRule.kMatchStep
    ef: EfSchedule = field(default_factory=EfSchedule)

    @staticmethod
    def from_json(doc) -> "CovapSettings":
        text = doc if isinstance(doc, str) else json.dumps(doc)
        c = L.SettingsC()
        L.lib().covap_settings_from_json(text.encode(), ctypes.byref(c))
        return CovapSettings._from_c(c)

    @staticmethod
    def _from_c(c) -> "CovapSettings":
        return CovapSettings(int(c.interval), bool(c.auto_interval), int(c.rule),
                             EfSchedule(bool(c.ef.enabled), c.ef.init_value, int(c.ef.ascend_steps),
                                        c.ef.ascend_range))

    def c(self):
        return L.SettingsC(int(self.interval), 1 if self.auto_interval else 0, int(self.rule),
                           self.ef.c())

    def resolve_interval(self, ccr_value: float) -> int:
        """resolve_interval (config.cpp:238-241)."""
        c, k = self.c(), ctypes.c_uint32()
        L.lib().covap_resolve_interval(ctypes.byref(c), float(ccr_value), ctypes.byref(k))
        return k.value

    def config(self, interval: Optional[int] = None) -> CovapConfig:
        """The CovapConfig of a run once K is known."""
        return CovapConfig(self.interval if interval is None else int(interval), self.rule, self.ef)


def settings_from_json(doc) -> CovapSettings:
    return CovapSettings.from_json(doc)


def resolve_interval(settings: CovapSettings, ccr_value: float) -> int:
    return settings.resolve_interval(ccr_value)


def ccr_decide(comm: Optional["Communicator"], own_comm_ms: Sequence[float],
               own_comp_ms: float) -> ProfileResult:
    """The live CCR controller in the library (covap_ccr_decide): rank-min of
    the per-collective arrival->completion durations over the communicator,
    rank 0's compute time, CCR and K — the same result on every rank."""
    n = len(own_comm_ms)
    d = (ctypes.c_double * max(n, 1))(*[float(x) for x in own_comm_ms])
    r = L.CcrResultC()
    L.lib().covap_ccr_decide(None if comm is None else comm.handle, d, n, float(own_comp_ms),
                             ctypes.byref(r))
    return ProfileResult(r.ccr, r.comp_ms, r.comm_aligned_ms,
                         [max(0.0, float(x)) for x in own_comm_ms], r.recommended_interval)


class CcrController:
    """CCR-driven choice of K (PAPER §IV-B; perf.cpp:40-53, sim.cpp:164-216).

    One dense iteration is profiled.  Each rank measures, per collective, the
    time from its own arrival to the collective's completion; the collective
    completes at the same instant everywhere, so the rank-minimum of those
    durations is ``end - last arrival`` — the reference's rendezvous-aligned
    communication time (sim.cpp:202-203) — without a global clock.  The
    compute time is worker 0's (sim.cpp:208-211).  Every rank then derives the
    same K = max(1, ceil(comm / comp))."""

    def __init__(self, exchange):
        self.exchange = exchange

    def decide(self, own_comm_ms: Sequence[float], own_comp_ms: float) -> ProfileResult:
        if isinstance(self.exchange, NcclExchange):  # all of it in the library
            return ccr_decide(self.exchange.comm, own_comm_ms, own_comp_ms)
        durs = [max(0.0, float(x)) for x in own_comm_ms]
        aligned, comp0 = self.exchange(durs, own_comp_ms)
        comm = float(sum(aligned))
        c = ccr(comm, comp0)
        return ProfileResult(c, comp0, comm, list(durs), choose_interval(c))


# ------------------------------------------------------------ peer collective

class PeerGroup:
    """C1 as a load/store collective over NVLink peer memory (covap_peer_*):
    the rank-ordered allreduce of the packed send buffers, bit-identical to
    allreduce_mean (trainer.cpp:41-43) for any P.  Rendezvous: every rank
    calls ``export()``, the blobs are gathered (torch.distributed), every
    rank calls ``import_(blobs)``; ranks of one process use ``attach_local``."""

    def __init__(self, state: CompressorState, nranks: int, rank: int, _handle=None):
        h = _handle
        if h is None:
            h = ctypes.c_void_p()
            L.lib().covap_peer_create(state.handle, int(nranks), int(rank), ctypes.byref(h))
        self._h = h
        self.state = state
        self.nranks, self.rank = int(nranks), int(rank)

    @staticmethod
    def from_nccl(state: CompressorState, comm: "Communicator", multimem: bool = False) -> "PeerGroup":
        """The buffers in an NCCL symmetric window on ``comm`` (no CUDA IPC
        rendezvous; collective over comm's ranks).  ``multimem``: reduce in
        the NVSwitch (multimem.ld_reduce / multimem.st) — switch summation
        order, the NCCL tolerance; raises where the communicator has no
        multicast.  Destroy the group before the communicator."""
        h = ctypes.c_void_p()
        L.lib().covap_peer_create_nccl(state.handle, comm.handle, int(bool(multimem)),
                                       ctypes.byref(h))
        g = PeerGroup(state, comm.nranks, comm.rank, _handle=h)
        g._comm = comm  # keep the communicator alive as long as the group
        return g

    @property
    def multimem(self) -> bool:
        on = ctypes.c_int32()
        L.lib().covap_peer_multimem(self._h, ctypes.byref(on))
        return bool(on.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._LIB is not None:
            L._LIB.covap_peer_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def export(self) -> bytes:
        n = ctypes.c_size_t()
        L.lib().covap_peer_export(self._h, None, 0, ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        L.lib().covap_peer_export(self._h, buf, n.value, ctypes.byref(n))
        return buf.raw

    def import_(self, blobs: Sequence[bytes]):
        blob = b"".join(blobs)
        L.lib().covap_peer_import(self._h, blob, len(blobs[0]))

    @staticmethod
    def attach_local(groups: Sequence["PeerGroup"]):
        arr = (ctypes.c_void_p * len(groups))(*[g.handle.value for g in groups])
        L.lib().covap_peer_attach_local(arr, len(groups))

    @staticmethod
    def from_torch_distributed(state: CompressorState) -> "PeerGroup":
        import torch.distributed as dist
        g = PeerGroup(state, dist.get_world_size(), dist.get_rank())
        blobs = [None] * dist.get_world_size()
        dist.all_gather_object(blobs, g.export())
        g.import_(blobs)
        return g

    def set_limits(self, max_ctas: int = 0, timeout_s: float = 0.0):
        L.lib().covap_peer_set_limits(self._h, int(max_ctas), float(timeout_s))

    MODE_GATHER, MODE_FUSED, MODE_STEP = 0, 1, 2

    def set_fused(self, fused):
        """True / 1: C1 + K2 in one kernel (default); False / 0: all-gather
        then K2; 2 (MODE_STEP): K1 + C1 + K2 as one kernel, chunk by chunk."""
        L.lib().covap_peer_set_fused(self._h, int(fused))

    def check(self):
        L.lib().covap_peer_check(self._h)

    def sync(self, grad, out, stream=None):
        """K1 -> peer allreduce (rank order) -> K2 x 1/P -> ++step."""
        self.state._check(grad)
        self.state._check(out)
        L.lib().covap_peer_sync_step(self.state.handle, self._h, _ptr(grad), _ptr(out),
                                     _stream_ptr(stream, self.state.device))


# ------------------------------------------------------------ timeline / overlap model

@dataclass
class OverlapSchedule:
    """OverlapSchedule (perf.hpp:40-58)."""
    total_ms: float
    stream_end_ms: float
    unoverlapped_comm_ms: float
    comm_start_ms: List[float]
    comm_end_ms: List[float]
    comm_tensor: List[int]
    bubbles: List[tuple]  # (after_tensor, duration_ms)


def overlap_schedule(before_ms: float, comp_ms: Sequence[float],
                     compress_ms: Optional[Sequence[float]], comm_ms: Sequence[float],
                     communicated: Optional[Sequence[bool]] = None) -> OverlapSchedule:
    """overlap_schedule (perf.cpp:63-103): the exact overlapped iteration."""
    n = len(comp_ms)
    if len(comm_ms) != n or (compress_ms is not None and len(compress_ms) != n) or \
            (communicated is not None and len(communicated) != n):
        raise InvalidInput("per-tensor lists have inconsistent lengths")
    dbl = ctypes.c_double * max(n, 1)
    c, m = dbl(*comp_ms), dbl(*comm_ms)
    cp = None if compress_ms is None else dbl(*compress_ms)
    sent = None if communicated is None else (ctypes.c_uint8 * max(n, 1))(*[1 if x else 0 for x in communicated])
    tot, se, un = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    cs, ce, bm = dbl(), dbl(), dbl()
    ct, ba = (ctypes.c_int64 * max(n, 1))(), (ctypes.c_int64 * max(n, 1))()
    nc, nb = ctypes.c_size_t(), ctypes.c_size_t()
    L.lib().covap_overlap_schedule(float(before_ms), c, cp, m, sent, n, ctypes.byref(tot),
                                   ctypes.byref(se), ctypes.byref(un), cs, ce, ct, ctypes.byref(nc),
                                   ba, bm, ctypes.byref(nb))
    k, b = nc.value, nb.value
    return OverlapSchedule(tot.value, se.value, un.value, list(cs[:k]), list(ce[:k]), list(ct[:k]),
                           [(ba[i], bm[i]) for i in range(b)])
