"""One rank of a multi-PROCESS COVAP sync run (tests/test_multiproc.py).

Launched P times (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the env),
every process on the same GPU (cuda:0 unless COVAP_MP_DEVICE is set) — the
one-GPU stand-in for one process per GPU.  Rendezvous over gloo
(torch.distributed is plumbing only); the data plane is the product's:

  --collective peer   PeerGroup.from_torch_distributed: covap_peer_export /
                      covap_peer_import over CUDA IPC, then covap_peer_sync_step
                      (modes 0/1/2) with st.release.sys / ld.acquire.sys flags
                      between PROCESSES;
  --collective nccl   Communicator.from_torch_distributed + covap_sync_step
                      (K1 -> ncclAllReduce -> K2; needs one GPU per rank).
  --collective peer_nccl  the peer kernels with their buffers in an NCCL
                      symmetric window (PeerGroup.from_nccl; --multimem: the
                      reduction in the NVSwitch); one GPU per rank.

Steps run back to back with no host synchronisation between them (the
schedule the ADVICE race needs: empty phases between same-parity steps), each
step's output copied aside on the stream.  Afterwards every rank checks its
outputs and its residual arena against the rank-ordered oracle restatement
(trainer.cpp:365-386; the oracle is the checker only) and writes a JSON
verdict to --out.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--interval", type=int, default=4)
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--collective", choices=["peer", "nccl", "peer_nccl"], default="peer")
    ap.add_argument("--multimem", action="store_true")
    ap.add_argument("--seed", type=int, default=21)
    ap.add_argument("--timeout", type=float, default=120.0)
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    verdict = {"rank": rank, "world": world, "ok": False}
    try:
        import numpy as np
        import torch
        import torch.distributed as dist

        import paper_2311_04499_b200 as covap
        from oracle.oracle import Oracle

        dev_index = int(os.environ.get("COVAP_MP_DEVICE", "-1"))
        if dev_index < 0:
            dev_index = rank if a.collective in ("nccl", "peer_nccl") else 0
        torch.cuda.set_device(dev_index)
        dev = torch.device("cuda", dev_index)
        dist.init_process_group("gloo", rank=rank, world_size=world)

        K = a.interval
        plan = covap.plan_for(covap.load_layout(a.layout), covap.CovapConfig(interval=K))
        ef = covap.EfSchedule(True, 0.3, 1, 0.2)
        d = plan.total_numel()
        stream = torch.cuda.Stream(dev)
        if a.collective == "peer":
            state = covap.CompressorState(plan, torch.float32, dev_index, ef)
            group = covap.PeerGroup.from_torch_distributed(state)
            group.set_limits(max_ctas=a.max_ctas, timeout_s=a.timeout)
            group.set_fused(a.mode)
            sync_fn = lambda g, o: group.sync(g, o, stream)  # noqa: E731
        elif a.collective == "peer_nccl":
            comm = covap.Communicator.from_torch_distributed(dev_index)
            state = covap.CompressorState(plan, torch.float32, dev_index, ef)
            group = covap.PeerGroup.from_nccl(state, comm, multimem=a.multimem)
            verdict["multimem"] = group.multimem
            group.set_limits(max_ctas=a.max_ctas, timeout_s=a.timeout)
            group.set_fused(a.mode)
            sync_fn = lambda g, o: group.sync(g, o, stream)  # noqa: E731
        else:
            comm = covap.Communicator.from_torch_distributed(dev_index)
            sync = covap.CovapSync(plan, comm, torch.float32, dev_index, ef)
            state = sync.state
            sync_fn = lambda g, o: sync.sync(g, o, stream)  # noqa: E731

        grads = []
        for s in range(a.steps):
            t = torch.empty(d, device=dev)
            covap.generate(t, covap.stream_key(a.seed, rank, s))
            grads.append(t)
        outs = [torch.empty(d, device=dev) for _ in range(a.steps)]
        out = torch.empty(d, device=dev)
        torch.cuda.synchronize(dev)
        dist.barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for s in range(a.steps):  # back to back: no host sync between steps
                sync_fn(grads[s], out)
                outs[s].copy_(out)
        stream.synchronize()
        verdict["wall_s"] = time.perf_counter() - t0
        if a.collective in ("peer", "peer_nccl"):
            group.check()  # raises if any spin-wait timed out
        got = [o.cpu().numpy() for o in outs]
        got_r = state.residuals.cpu().numpy()
        dist.barrier()

        # ---- the checker: every rank's K1 in rank order, then the mean ----
        orc = Oracle()
        tensors = [(t.bucket, t.begin, t.end) for t in plan.tensors]
        rs = [np.zeros(d, np.float32) for _ in range(world)]
        mism = []
        for s in range(a.steps):
            keep = orc.select(s, K, len(tensors))
            coeff = np.float32(orc.ef_coefficient(s, 0.3, 1, 0.2))
            pays = [orc.compress(orc.generate(orc.stream_key(a.seed, w, s), d, 0, 0, np.float32),
                                 rs[w], tensors, keep, 1, coeff) for w in range(world)]
            mean = orc.allreduce_mean(np.stack(pays)) if len(pays[0]) else pays[0]
            want = orc.decompress(mean, tensors, keep, d, np.float32)
            if (a.collective == "nccl" and world > 2) or (a.multimem and world > 1):
                # NCCL's (or the NVSwitch's) summation order differs from the
                # rank order: the stated bound |d| <= 1e-6 * sum_w |x_w|
                absx = orc.decompress(np.sum(np.abs(np.stack(pays)).astype(np.float64), axis=0),
                                      tensors, keep, d, np.float64)
                bad = np.abs(got[s].astype(np.float64) - want) > 1e-6 * absx / world + 0.0
                n_bad = int(bad.sum())
            else:
                n_bad = int((got[s].view(np.uint32) != want.view(np.uint32)).sum())
            if n_bad:
                mism.append({"step": s, "out_mismatches": n_bad})
        n_bad_r = int((got_r.view(np.uint32) != rs[rank].view(np.uint32)).sum())
        if n_bad_r:
            mism.append({"residual_mismatches": n_bad_r})
        verdict.update(ok=not mism, mismatches=mism, elements=d,
                       selected_per_step=[int(plan.send_elems(s)[1]) for s in range(a.steps)])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported through the verdict file
        import traceback
        verdict["error"] = f"{type(e).__name__}: {e}"
        verdict["trace"] = traceback.format_exc()[-2000:]
    with open(a.out, "w") as f:
        json.dump(verdict, f)
    os._exit(0 if verdict["ok"] else 1)  # no atexit teardown of IPC mappings mid-peer-read


if __name__ == "__main__":
    main()
