"""Probe K2 timing in isolation vs right after K1 (not product code)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2311_04499_b200 as covap

def ev():
    return torch.cuda.Event(enable_timing=True)

for name, K in (("resnet50", 4), ("resnet50", 1), ("bert_large", 4)):
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    st = covap.CompressorState(plan, torch.float32, 0)
    n = plan.total_numel()
    g = torch.empty(n, device="cuda"); covap.generate(g, 5)
    out = torch.empty(n, device="cuda")
    for phase in range(K):
        st.num_steps = phase
        _, S = plan.send_elems(phase)
        byt = 4 * n + 4 * S
        # K2 alone, back to back
        for _ in range(3): st.unpack(out, 1.0, True)
        e0, e1 = ev(), ev(); e0.record()
        for _ in range(10): st.unpack(out, 1.0, True)
        e1.record(); torch.cuda.synchronize()
        t_alone = e0.elapsed_time(e1) / 10
        # K1 then K2
        tk2 = 0.0
        for i in range(10):
            st.num_steps = phase
            st.filter_pack(g)
            a, b = ev(), ev(); a.record(); st.unpack(out, 1.0, True); b.record()
            torch.cuda.synchronize(); tk2 += a.elapsed_time(b)
        tk2 /= 10
        print(f"{name} K{K} phase {phase} S={S}: K2 alone {t_alone*1e3:.1f} us ({byt/t_alone/1e6:.0f} GB/s)  after K1 {tk2*1e3:.1f} us ({byt/tk2/1e6:.0f} GB/s)")
