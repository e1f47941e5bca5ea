"""COVAP vs the baseline compressors on one B200.

For one layout, times one synchronisation step per scheme on the device
(inputs resident, back to back, CUDA events, inputs larger than L2):
  covap     K1F fused pass (CovapSync, one rank)           trainer.cpp:365-386
  topk      ErrorFeedback + TopkFilter(k) + exchange/mean  trainer.cpp:387-403
  randomk   ErrorFeedback + RandomkFilter(k, seed) + mean
  fp16      ErrorFeedback + Fp16Filter + mean
and, for the same scheme, the reference's own CPU ErrorFeedback::step /
covap_compress (oracle/_ref, single-threaded as shipped) on the same layout,
bounded to --cpu-steps steps.  Prints one JSON line per scheme.

    python scripts/bench_baselines.py --layout resnet50 --k-fraction 0.01
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--k-fraction", type=float, default=0.01)
    ap.add_argument("--interval", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--schemes", default="covap,topk,randomk,fp16")
    ap.add_argument("--breakdown", action="store_true", help="per-phase event times (top-k)")
    args = ap.parse_args()

    import torch
    import paper_2311_04499_b200 as c
    from paper_2311_04499_b200 import feedback as F

    dev = torch.device("cuda", 0)
    model = c.load_layout(args.layout)
    buckets = [b.numel for b in c.allocate_buckets(model).buckets]
    n = sum(buckets)
    grads = []
    for s in range(3):  # rotate: 3 x (g) plus state > L2 (126 MB) at R50 size and up
        g = torch.empty(n, dtype=torch.float32, device=dev)
        c.generate(g, c.stream_key(1, 0, s), 0)
        grads.append(g)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    ef = c.EfSchedule()

    ref = None
    try:
        from oracle.oracle import Ref, RefFeedback, RefSession
        ref = Ref()
    except Exception as e:  # reference not built on this host
        print(f"[bench_baselines] reference arm unavailable: {e}", file=sys.stderr)

    for scheme in args.schemes.split(","):
        if scheme == "covap":
            plan = c.plan_for(model, c.CovapConfig(interval=args.interval))
            sync = c.CovapSync(plan, None)
            step = lambda g: sync.sync(g, out)  # noqa: E731
            wire = lambda: 4 * plan.payload_elements(0)  # noqa: E731
            kind = 1
        else:
            flt = {"topk": F.TopkFilter(args.k_fraction),
                   "randomk": F.RandomkFilter(args.k_fraction, 1),
                   "fp16": F.Fp16Filter()}[scheme]
            fb = F.ErrorFeedback(buckets, ef, flt)
            step = lambda g, fb=fb: fb.sync(g, out)  # noqa: E731
            wire = lambda fb=fb: fb.wire_bytes()  # noqa: E731
            kind = flt.kind
        for i in range(args.warmup):
            step(grads[i % 3])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            step(grads[i % 3])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        line = {"layout": args.layout, "scheme": scheme, "n": n, "buckets": len(buckets),
                "k_fraction": args.k_fraction if scheme in ("topk", "randomk") else None,
                "interval": args.interval if scheme == "covap" else None,
                "ms_per_step": round(ms, 4), "dense_equiv_GBps": round(4 * n / ms / 1e6, 1),
                "wire_bytes_per_step": int(wire())}
        if ref is not None and args.cpu_steps > 0:
            gh = [grads[i % 3].double().cpu().numpy() for i in range(args.cpu_steps)]
            if scheme == "covap":
                rs = RefSession(ref, [t.numel() for t in plan.tensors], 1, args.interval)
                secs = [rs.step(g)[2] for g in gh]
                rs.close()
            else:
                rf = RefFeedback(ref, buckets, kind, k_fraction=args.k_fraction, seed=1)
                secs = [rf.step(g)[3] for g in gh]
                rf.close()
            line["reference_cpu_ms_per_step"] = round(1e3 * float(np.mean(secs)), 2)
            line["reference_cpu_steps"] = len(secs)
            line["speedup_vs_reference_cpu"] = round(line["reference_cpu_ms_per_step"] / ms, 1)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
