"""K2 (unpack) on the BASELINE config-5 layout (16 equal buckets of B MB) at
interval K, a few back-to-back launches — for ncu (not product code)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=1)
ap.add_argument("--interval", type=int, default=2)
ap.add_argument("--iters", type=int, default=4)
a = ap.parse_args()
elems = a.mb * (1 << 20) // 4
model = covap.ModelSpec([covap.LayerSpec(f"l{i}", elems) for i in range(16)], bucket_cap_bytes=a.mb << 20)
plan = covap.plan_for(model, covap.CovapConfig(interval=a.interval))
n = plan.total_numel()
out = torch.empty(n, device="cuda")
st = covap.CompressorState(plan, torch.float32, 0)
for _ in range(a.iters):
    st.unpack(out, 1.0, True)
torch.cuda.synchronize()
print("ok", n)
