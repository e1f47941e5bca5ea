"""K1F (one-rank sync step) timing three ways (probe, not product):
eager back to back from e_first (the bench's loop), the same behind a
head-start spin, and one K-cycle captured in a CUDA graph and replayed."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

PEAK = 6531.3


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for name, K in (("resnet50", 4), ("resnet50", 1), ("bert_large", 4)):
        plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
        sync = covap.CovapSync(plan, None, torch.float32, 0)
        st = sync.state
        n = plan.total_numel()
        grads = [torch.empty(n, device=dev) for _ in range(3)]
        for i, g in enumerate(grads):
            covap.generate(g, covap.stream_key(1, 0, i))
        out = torch.empty(n, device=dev)
        steps = 40
        for s in range(8):
            sync.sync(grads[s % 3], out)
        torch.cuda.synchronize()
        res = {"layout": name, "K": K}
        for mode in ("eager", "eager_headstart"):
            a, b = ev(), ev()
            if mode == "eager_headstart":
                covap.spin(300.0, 1, stream)
            a.record(stream)
            for s in range(steps):
                sync.sync(grads[s % 3], out)
            b.record(stream)
            torch.cuda.synchronize()
            res[mode + "_us"] = round(a.elapsed_time(b) / steps * 1e3, 2)
        cap = torch.cuda.Stream(dev)
        gr = torch.cuda.CUDAGraph()
        base = st.num_steps
        with torch.cuda.stream(cap):
            with torch.cuda.graph(gr, stream=cap):
                for k in range(K * 3):
                    sync.sync(grads[k % 3], out)
        st.num_steps = base
        gr.replay()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        reps = max(1, steps // (3 * K))
        a.record(stream)
        for _ in range(reps):
            gr.replay()
        b.record(stream)
        torch.cuda.synchronize()
        res["graph_us"] = round(a.elapsed_time(b) / (reps * 3 * K) * 1e3, 2)
        for k in ("eager_us", "eager_headstart_us", "graph_us"):
            res[k.replace("_us", "_frac")] = round(16 * n / (res[k] * 1e-6) / 1e9 / PEAK, 4)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
