"""PCIe and host-pipeline chunk-schedule probe (not product code)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2311_04499_b200 as covap

n = 25557032
hin = torch.empty(n, pin_memory=True); hout = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
h2d = t(lambda: d1.copy_(hin, non_blocking=True))
d2h = t(lambda: hout.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2): hout.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bb = t(both)
B = 4 * n / 1e9
print(f"H2D {h2d:.3f} ms ({B/h2d*1e3:.1f} GB/s)  D2H {d2h:.3f} ms ({B/d2h*1e3:.1f} GB/s)  both concurrently {bb:.3f} ms")
for name in ("resnet50", "bert_large"):
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=1))
    n = plan.total_numel()
    hin = torch.empty(n, pin_memory=True); hout = torch.empty(n, pin_memory=True)
    sync = covap.CovapSync(plan, None, torch.float32, 0)
    for chunk in (1 << 21, 1 << 22, 1 << 23, 3 << 22):
        for ramp in (1 << 20, 1 << 18, 1 << 16, 1 << 14):
            if ramp >= chunk // 2 and ramp != 1 << 20:
                continue
            sync.state.set_host_ramp(ramp)
            ms = t(lambda: sync.sync_host(hin, hout, chunk_elems=chunk), reps=5 if name == "bert_large" else 10)
            print(f"{name} chunk {chunk / (1 << 20):g} Mi ramp_min {ramp / (1 << 10):g} Ki: {ms:.3f} ms -> e2e {4*n/ms/1e6:.1f} GB/s",
                  flush=True)
