"""COVAP as a PyTorch DDP communication hook — the paper's integration point
(SURVEY.md §8(f) rank 1).

DDP hands the hook one ``GradBucket`` at a time, in bucket index order, as
backward produces them.  The hook runs the B200 path on the bucket's own
buffer: K1 (filter_pack) on the producing stream, the allreduce of the
bucket's selected shard and K2 (unpack, x1/P) on the side stream
(``covap_bucket_ready_local``); the future the hook returns is CUDA-aware and
completes on the stream that finishes the bucket, so DDP's wait orders its
use of the bucket after the unpack; the last bucket closes the step
(``covap_step_finish``).  DDP's buckets are the reference's buckets: the plan
is built with one "layer" per DDP bucket and a 1-byte cap, so
``allocate_buckets`` reproduces them and the median / sharding / selection
rules (model.cpp:66-115, compress.cpp:13-28) apply to them unchanged; the
plan is padded so every bucket buffer can stand for its slice of the arena.

DDP may rebuild its buckets after the first iteration, so the hook observes
``warmup`` iterations with the plain allreduce-mean (dense) before it builds
the plan and switches to COVAP.

    model = DDP(net, bucket_cap_mb=25, gradient_as_bucket_view=True)
    hook = CovapDDPHook(covap.CovapConfig(interval=K), comm)
    model.register_comm_hook(hook, CovapDDPHook.hook)
"""
from __future__ import annotations

from typing import List, Optional

from .covap import BucketPlan, Communicator, CovapConfig, CovapSync, LayerSpec, ModelSpec


def _torch():
    import torch
    return torch


class CovapDDPHook:
    """State object for ``DistributedDataParallel.register_comm_hook``."""

    def __init__(self, config: CovapConfig, comm: Optional[Communicator] = None,
                 device: Optional[int] = None, warmup: int = 2, fuse_single_rank: bool = True,
                 free_sms: int = 0):
        torch = _torch()
        self.config = config
        self.comm = comm
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.warmup = int(warmup)
        # one rank: the fused K1F pass on the producing stream (default), or the
        # multi-rank schedule (K1 here, allreduce + unpack on the side stream)
        self.fuse_single_rank = bool(fuse_single_rank)
        # SMs the multi-rank schedule's K1 / K2 leave to the allreduce kernels
        self.free_sms = int(free_sms)
        self.sync: Optional[CovapSync] = None
        self.plan: Optional[BucketPlan] = None
        self.iterations = 0
        self._sizes: List[int] = []
        self._prev_sizes: List[int] = []
        self.bucket_params: List[list] = []  # parameter lists per bucket (last observed)

    @property
    def world(self) -> int:
        return self.comm.nranks if self.comm is not None else 1

    # -- dense warm-up ----------------------------------------------------
    def _dense(self, bucket):
        torch = _torch()
        buf = bucket.buffer()
        if self.comm is not None and self.comm.nranks > 1:
            self.comm.allreduce(buf)
        buf.mul_(1.0 / self.world)
        fut = torch.futures.Future()
        fut.set_result(buf)
        return fut

    def _build(self):
        model = ModelSpec([LayerSpec(f"ddp_bucket{i}", int(n)) for i, n in enumerate(self._sizes)],
                          bucket_cap_bytes=1)
        self.plan = BucketPlan(model, None, interval=self.config.interval, rule=self.config.rule,
                               shard=-1, pad=True)
        assert [b.numel for b in self.plan.buckets] == self._sizes
        self.sync = CovapSync(self.plan, self.comm, _torch().float32, self.device, self.config.ef,
                              fuse_single_rank=self.fuse_single_rank, free_sms=self.free_sms)
        self._side = self.sync.side_stream()

    # -- the hook ---------------------------------------------------------
    @staticmethod
    def hook(state: "CovapDDPHook", bucket):
        torch = _torch()
        idx = bucket.index()
        buf = bucket.buffer()
        if state.sync is None:
            if idx == 0:
                state._sizes = []
                state.bucket_params = []
            state._sizes.append(buf.numel())
            state.bucket_params.append(list(bucket.parameters()))
            fut = state._dense(bucket)
            if bucket.is_last():
                state.iterations += 1
                stable = state._sizes == state._prev_sizes
                state._prev_sizes = list(state._sizes)
                if state.iterations >= state.warmup and stable:
                    state._build()
            return fut
        if buf.dtype != torch.float32 or not buf.is_contiguous():
            raise TypeError("the COVAP hook handles contiguous fp32 gradient buckets")
        stream = torch.cuda.current_stream(state.device)
        state.sync.bucket_ready_local(idx, buf, buf, stream)
        # A CUDA-aware future completed on the stream that finishes this
        # bucket: DDP's wait() makes its stream wait for this bucket's unpack
        # (side stream) or fused pass (producing stream) — nothing here relies
        # on finish() ordering the streams.
        fut = torch.futures.Future(devices=[torch.device("cuda", state.device)])
        if state.world == 1 and state.fuse_single_rank:
            fut.set_result(buf)
        else:
            with torch.cuda.stream(state._side):
                fut.set_result(buf)
        if bucket.is_last():
            state.sync.finish(stream)
            state.iterations += 1
        return fut
