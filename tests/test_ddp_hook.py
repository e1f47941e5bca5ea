"""The DDP communication-hook adapter on a B200:
real backward passes drive the COVAP schedule through DistributedDataParallel
(world size 1, NCCL backend) and the synchronised gradients DDP hands to the
optimizer equal the fp32 oracle applied to the raw bucket gradients, bit for
bit, step after step (residuals carried)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("K,schedule,view", [(1, "fused", True), (3, "fused", True),
                                             (3, "side", True), (3, "side", False),
                                             (1, "side", False), (3, "fused", False)])
def test_ddp_hook_matches_oracle(pg, covap, orc, K, schedule, view):
    """schedule 'fused': one rank's K1F on the producing stream; 'side': the
    multi-rank schedule through a 1-rank NCCL communicator (K1 with the zero
    fill on the producing stream, allreduce + selected-only unpack on the
    side stream, finish() joins the streams).  view False: DDP copies the
    bucket back into .grad after the hook's future — the copy must see the
    side-stream unpack."""
    from torch.nn.parallel import DistributedDataParallel as DDP
    from paper_2311_04499_b200.ddp import CovapDDPHook
    torch.manual_seed(0)
    net = torch.nn.Sequential(
        torch.nn.Linear(256, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 4096), torch.nn.ReLU(),
        torch.nn.Linear(4096, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 64)).cuda()
    model = DDP(net, bucket_cap_mb=4, gradient_as_bucket_view=view)
    ef = covap.EfSchedule(True, 0.5, 1, 0.25)
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0) if schedule == "side" else None
    hook = CovapDDPHook(covap.CovapConfig(interval=K, ef=ef), comm, 0, warmup=2,
                        fuse_single_rank=schedule == "fused")
    raw = {}

    def spy(state, bucket):  # the bucket's local gradient before COVAP touches it
        raw[bucket.index()] = bucket.buffer().detach().clone()
        return CovapDDPHook.hook(state, bucket)

    model.register_comm_hook(hook, spy)
    x = torch.randn(32, 256, device="cuda")
    for it in range(5):  # DDP may rebuild buckets after the first iteration
        model(x).square().mean().backward()
        model.zero_grad(set_to_none=False)
        if hook.sync is not None:
            break
    assert hook.sync is not None, (hook.iterations, hook._sizes, hook._prev_sizes)
    assert len(hook.plan.buckets) >= 3
    plan = hook.plan
    tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
    d = plan.total_numel()
    r = np.zeros(d, np.float32)
    for s in range(2 * K + 1):
        raw.clear()
        model(x * (1 + s)).square().mean().backward()
        torch.cuda.synchronize()
        g = np.concatenate([raw[b].cpu().numpy() for b in range(len(plan.buckets))])
        keep = orc.select(s, K, len(tensors))
        p = orc.compress(g, r, tensors, keep, 1, np.float32(orc.ef_coefficient(s, 0.5, 1, 0.25)))
        want = orc.decompress(orc.allreduce_mean(p[None, :]) if len(p) else p, tensors, keep, d,
                              np.float32)
        # DDP's gradients (views of the bucket buffers) after the hook
        got = np.concatenate([torch.cat([q.grad.reshape(-1) for q in ps]).cpu().numpy()
                              for ps in hook.bucket_params])
        assert np.array_equal(bits(got), bits(want)), s
        res = hook.sync.state.residuals.cpu().numpy()
        dev = np.concatenate([res[plan.device_begin(b):plan.device_begin(b) + plan.buckets[b].numel]
                              for b in range(len(plan.buckets))])
        assert np.array_equal(bits(dev), bits(r)), s
        model.zero_grad(set_to_none=False)
    if comm is not None:
        comm.close()
