"""Kernel timeline of back-to-back baseline-compressor sync steps (CUPTI via
torch.profiler; not product code).  Prints, per kernel, start / end relative
to the first kernel of the last steps, so side-stream overlap is visible.

    python scripts/kernel_timeline.py --layout resnet50 --scheme randomk --steps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2311_04499_b200 as c  # noqa: E402
from paper_2311_04499_b200 import feedback as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="resnet50")
ap.add_argument("--scheme", default="randomk")
ap.add_argument("--k-fraction", type=float, default=0.01)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()

dev = torch.device("cuda", 0)
buckets = [b.numel for b in c.allocate_buckets(c.load_layout(a.layout)).buckets]
n = sum(buckets)
grads = []
for s in range(3):
    g = torch.empty(n, dtype=torch.float32, device=dev)
    c.generate(g, c.stream_key(1, 0, s), 0)
    grads.append(g)
out = torch.empty(n, dtype=torch.float32, device=dev)
flt = {"topk": F.TopkFilter(a.k_fraction), "randomk": F.RandomkFilter(a.k_fraction, 1),
       "fp16": F.Fp16Filter()}[a.scheme]
fb = F.ErrorFeedback(buckets, c.EfSchedule(), flt)
for i in range(6):
    fb.sync(grads[i % 3], out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(a.steps):
        fb.sync(grads[i % 3], out)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    name = e.name.split("(")[0].replace("void ", "")[-48:]
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:7.1f}"
          f"  s{getattr(e, 'device_resource_id', '?')}  {name}")
span = ev[-1].time_range.end - t0
print(f"span {span:.1f} us for {a.steps} steps: {span / a.steps:.1f} us/step")
