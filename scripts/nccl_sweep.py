"""C1 characterisation at P ranks (BASELINE config 5, the allreduce half):
bus bandwidth of the selected-shard allreduce through the library's NCCL
communicator (covap_allreduce, sum, fp32) for messages of 1 MB - 1 GB, and
of the whole multi-rank sync step (K1 -> allreduce -> K2, covap_sync_step)
on the synthetic 16-bucket layouts at K = 1 / 4.  One process per GPU:

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        scripts/nccl_sweep.py --out gpurun_out/nccl_sweep.jsonl

Bus bytes = 2(P-1)/P x message bytes (the ring volume, sim.cpp:28-35),
against 900 GB/s per direction per GPU (NVLink 5).  Times are CUDA events
on the launching stream, max over ranks.  At P = 1 there is nothing to
measure (the allreduce of one rank is the identity) and the script says so.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2311_04499_b200 as covap

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:
        print(json.dumps({"P": 1, "note": "one rank: the allreduce is the identity, no bus traffic"}))
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", device_id=dev)
    comm = covap.Communicator.from_torch_distributed(local)
    stream = torch.cuda.current_stream(dev)
    lines = []

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    mb = 1
    while mb <= a.max_mb:
        n = mb * (1 << 20) // 4
        buf = torch.ones(n, device=dev)
        ms = timed(lambda: comm.allreduce(buf, stream), a.reps)
        bus = 2.0 * (world - 1) / world * 4 * n
        lines.append({"what": "allreduce", "P": world, "mb": mb, "ms": round(ms, 5),
                      "bus_gbs": round(bus / (ms * 1e-3) / 1e9, 1),
                      "frac_of_900": round(bus / (ms * 1e-3) / 1e9 / 900.0, 4)})
        del buf
        # the whole multi-rank step on 16 buckets of mb / 16 MB each
        if mb >= 16:
            elems = n // 16
            model = covap.ModelSpec([covap.LayerSpec(f"l{i}", elems) for i in range(16)],
                                    bucket_cap_bytes=elems * 4)
            for K in (1, 4):
                plan = covap.plan_for(model, covap.CovapConfig(interval=K))
                sync = covap.CovapSync(plan, comm, torch.float32, local)
                g = torch.empty(plan.device_numel(), device=dev)
                covap.generate(g, covap.stream_key(1, rank, 0))
                out = torch.empty_like(g)
                ms = timed(lambda: sync.sync(g, out, stream), max(K, a.reps // K * K))
                lines.append({"what": "sync_step", "P": world, "mb": mb, "K": K,
                              "ms": round(ms, 5),
                              "sync_gbs_per_gpu": round(4 * 16 * elems / (ms * 1e-3) / 1e9, 1)})
                del sync, g, out
        torch.cuda.empty_cache()
        mb *= 2
    if rank == 0:
        for l in lines:
            print(json.dumps(l), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                f.write("\n".join(json.dumps(l) for l in lines) + "\n")
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
