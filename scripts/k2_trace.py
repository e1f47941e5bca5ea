"""Per-CTA timeline of K2 (diagnostic build with -DCOVAP_K2_TRACE; not product code).

    COVAP_LIB_PATH=.../_variants/k2trace/libcovap_b200.so python scripts/k2_trace.py --mb 1 --interval 2
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402
from paper_2311_04499_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=1)
ap.add_argument("--interval", type=int, default=2)
ap.add_argument("--layout", default=None)
a = ap.parse_args()
if a.layout:
    model = covap.load_layout(a.layout)
else:
    elems = a.mb * (1 << 20) // 4
    model = covap.ModelSpec([covap.LayerSpec(f"l{i}", elems) for i in range(16)], bucket_cap_bytes=a.mb << 20)
plan = covap.plan_for(model, covap.CovapConfig(interval=a.interval))
n = plan.total_numel()
out = torch.empty(n, device="cuda")
st = covap.CompressorState(plan, torch.float32, 0)
lib = L.lib()
fn = lib.dll.covap_debug_k2_trace
for ph in range(a.interval):
    for _ in range(3):
        st.num_steps = ph
        st.unpack(out, 1.0, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.unpack(out, 1.0, True)
    e1.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (148 * 6))()
    fn(buf, 148)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 6).astype(np.int64)
    t0 = t[:, 0].min()
    dur = (t[:, 1] - t[:, 0]) / 1e3
    print(f"phase {ph}: event {e0.elapsed_time(e1)*1e3:.1f} us; CTA start spread {(t[:,0].max()-t0)/1e3:.1f} us, "
          f"end max {(t[:,1].max()-t0)/1e3:.1f} us; CTA dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
    i = int(np.argmax(dur))
    print(f"  slowest CTA {i}: full {t[i,2]} none {t[i,3]} mixed {t[i,4]} wait {t[i,5]/1e3:.1f} us; "
          f"tiles full/none/mixed totals {t[:,2].sum()}/{t[:,3].sum()}/{t[:,4].sum()}; mean wait {t[:,5].mean()/1e3:.1f} us")
    for q in np.argsort(-dur)[:5]:
        print(f"   cta {q}: dur {dur[q]:.1f} full {t[q,2]} none {t[q,3]} mixed {t[q,4]} wait {t[q,5]/1e3:.1f}")
