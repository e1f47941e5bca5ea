"""A few whole-step peer launches (mode 2) at P = 1 for ncu (not product code)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=K))
st = covap.CompressorState(plan, torch.float32, 0)
grp = covap.PeerGroup(st, 1, 0)
covap.PeerGroup.attach_local([grp])
grp.set_fused(2)
d = plan.total_numel()
g = torch.empty(d, device="cuda")
covap.generate(g, covap.stream_key(1, 0, 0))
out = torch.empty(d, device="cuda")
for _ in range(4):
    grp.sync(g, out)
torch.cuda.synchronize()
grp.check()
print("ok")
