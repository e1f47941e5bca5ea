"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

* every rank builds its plan / selection independently and they agree
  (selection needs no communication, test_compress.cpp:94-101);
* the CCR controller's exchange (rank-min of own durations + rank 0's compute
  time) gives every rank the same K, equal to the reference's profile_ccr on
  the gathered traces (sim.cpp:164-216);
* the per-rank decomposition the GPU path uses — K1 on each rank, a SUM
  allreduce of the packed payload, K2 with x 1/P — reproduces the reference's
  in-process step (trainer.cpp:365-386) bit-for-bit at P = 2 (the oracle plays
  K1/K2 here; gloo plays NCCL).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import json
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2311_04499_b200 as covap
        from oracle.oracle import Oracle
        orc = Oracle()

        # 1. independent plans/selections agree
        digests = []
        for name, K in (("resnet50", 4), ("vgg16", 8), ("bert_large", 4)):
            p = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
            digests.append([(t.begin, t.end) for t in p.tensors])
            digests.append([p.selection(s) for s in range(3 * K)])
        gathered = [None] * world
        dist.all_gather_object(gathered, digests)
        assert all(g == gathered[0] for g in gathered)

        # 2. CCR controller: rank 1 arrives late at collective 1
        arrive = [[0.0, 10.0, 30.0], [0.0, 25.0, 30.0]][rank]
        end = [5.0, 40.0, 33.0]
        own = [e - a for e, a in zip(end, arrive)]
        comp = [50.0, 47.0][rank]
        res = covap.CcrController(covap.covap.TorchDistExchange()).decide(own, comp)
        ref = covap.profile_ccr([[0.0, 10.0, 30.0], [0.0, 25.0, 30.0]], end, 50.0, 2)
        assert res.comm_aligned_ms == ref.comm_aligned_ms == 5.0 + 15.0 + 3.0
        assert res.comp_ms == 50.0 and res.recommended_interval == ref.recommended_interval == 1
        ks = [None] * world
        dist.all_gather_object(ks, (res.ccr, res.recommended_interval))
        assert ks[0] == ks[1]
        big = covap.CcrController(covap.covap.TorchDistExchange()).decide([x * 10 for x in own], comp)
        assert big.recommended_interval == covap.choose_interval(230.0 / 50.0) == 5

        # 3. per-rank decomposition == reference in-process step (P = 2)
        with open(os.path.join(GOLDEN, "manifest.json")) as f:
            case = [c for c in json.load(f)["session"] if c["P"] == 2][0]
        fx = np.load(os.path.join(GOLDEN, f"session_{case['name']}.npz"))
        _, tensors = orc.plan(case["sizes"], case["cap"], case["K"])
        d = tensors[-1][2]
        r = np.zeros(d)
        en, init, asc, rng = case["ef"]
        for s in range(case["steps"]):
            keep = orc.select(s, case["K"], len(tensors), case["rule"])
            g = orc.generate(orc.stream_key(case["seed"], rank, s), d, case["kind"], 0, np.float64)
            payload = orc.compress(g, r, tensors, keep, en, orc.ef_coefficient(s, init, asc, rng))
            t = torch.from_numpy(payload.copy())
            if t.numel():
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
            mean = (0.0 + t.numpy()) * (1.0 / world)
            upd = orc.decompress(mean, tensors, keep, d, np.float64)
            assert np.array_equal(upd, fx[f"update_{s}"]), s
            if rank == 0:
                assert np.array_equal(r, fx[f"residual0_{s}"])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
