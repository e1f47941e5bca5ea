"""Run only the sync kernels of one layout, for ncu (not product code).

    python scripts/profile_step.py --layout resnet50 --interval 1 --mode fused --iters 6
modes: fused (K1F), unfused (the multi-rank kernels: K1 with the output zero
fill, then the selected-only K2).  L2 is flushed before every step.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="resnet50")
ap.add_argument("--interval", type=int, default=1)
ap.add_argument("--mode", default="fused", choices=["fused", "unfused"])
ap.add_argument("--iters", type=int, default=6)
a = ap.parse_args()
plan = covap.plan_for(covap.load_layout(a.layout), covap.CovapConfig(interval=a.interval))
st = covap.CompressorState(plan, torch.float32, 0)
n = plan.total_numel()
g = torch.empty(n, device="cuda")
out = torch.empty(n, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
for s in range(a.iters):
    covap.generate(g, covap.stream_key(1, 0, s))
    flush.zero_()
    if a.mode == "fused":
        st.filter_unpack(g, out)
    else:
        st.filter_pack(g, out=out)
        st.unpack(out, 1.0, True, selected_only=True)
    st.step_end()
torch.cuda.synchronize()
print("done", a)
