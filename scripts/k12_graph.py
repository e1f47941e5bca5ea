"""Graph-timed K1 (filter_pack + output zero fill, 16N) and K2 (selected-only
unpack, 8S) of the multi-rank sync step on BASELINE layouts: the whole layout
per step (covap_sync_step's kernels) and bucket by bucket (covap_bucket_ready's
kernels in the overlapped schedule).  One K-cycle per CUDA graph, replayed.

    python scripts/k12_graph.py [--layouts resnet50:4,bert_large:4] [--label base]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layouts", default="resnet50:4,resnet50:1,vgg16:4,bert_large:4")
ap.add_argument("--label", default="")
a = ap.parse_args()
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
    peak = json.load(f)["hbm_gbs"]


def graph_ms(fn, K, reps):
    cap = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        fn(0)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=cap):
            for k in range(K):
                fn(k)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps  # per K-cycle


for item in a.layouts.split(","):
    name, K = item.split(":")
    K = int(K)
    plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
    st = covap.CompressorState(plan, torch.float32, 0)
    n = plan.total_numel()
    grads = [torch.empty(n, device="cuda") for _ in range(3)]
    for i, g in enumerate(grads):
        covap.generate(g, covap.stream_key(1, 0, i))
    out = torch.empty(n, device="cuda")
    nb = len(plan.buckets)
    S = [plan.send_elems(s)[1] for s in range(K)]
    reps = 20

    def k1(k):
        st.num_steps = k
        st.filter_pack(grads[k % 3], out=out)

    def k2(k):
        st.num_steps = k
        st.unpack(out, 0.5, True, selected_only=True)

    def k1b(k):
        st.num_steps = k
        for b in range(nb):
            st.filter_pack(grads[k % 3], b, b + 1, out=out)

    def k2b(k):
        st.num_steps = k
        for b in range(nb):
            st.unpack(out, 0.5, True, b, b + 1, selected_only=True)

    t1, t2 = graph_ms(k1, K, reps), graph_ms(k2, K, reps)
    t1b, t2b = graph_ms(k1b, K, reps), graph_ms(k2b, K, reps)
    b1, b2 = 16 * n * K, 8 * sum(S)
    fr = lambda b, t: round(b / (t * 1e-3) / 1e9 / peak, 4)  # noqa: E731
    print(json.dumps({"label": a.label, "layout": name, "K": K, "buckets": nb,
                      "k1_us": round(t1 * 1e3 / K, 2), "k1_frac": fr(b1, t1),
                      "k2_us": round(t2 * 1e3 / K, 2), "k2_frac": fr(b2, t2),
                      "k1k2_frac": fr(b1 + b2, t1 + t2),
                      "per_bucket_k1_frac": fr(b1, t1b), "per_bucket_k2_frac": fr(b2, t2b),
                      "per_bucket_k2_us_per_step": round(t2b * 1e3 / K, 2)}), flush=True)
    del st, grads, out
    torch.cuda.empty_cache()
