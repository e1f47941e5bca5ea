"""BASELINE config 5: synthetic bucket sweep, 1 MB - 1 GB buckets x K in
{1, 2, 4, 8, 16} (kernel roofline characterisation, one GPU).

Layout per point: 16 equal layers of B bytes with a B-byte bucket cap, so 16
unsharded buckets and S = N/K exactly for every K dividing 16 (SURVEY.md
§8(d)).  Per point: the fused single-rank sync (K1F) and the multi-rank
kernels K1 and K2, timed back to back over whole K-cycles with CUDA events
(gradients rotate over 3 pre-generated buffers when they fit, so inputs
exceed L2 at every size from 16 MB up).  Writes a markdown table.

    python scripts/sweep.py [--max-mb 1024] [--out gpurun_out/sweep.md]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-mb", type=int, default=1024)
ap.add_argument("--min-mb", type=int, default=1)
ap.add_argument("--out", default="gpurun_out/sweep.md")
a = ap.parse_args()
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
    peak = json.load(f)["hbm_gbs"]

rows = []
mb = a.min_mb
while mb <= a.max_mb:
    elems = mb * (1 << 20) // 4
    model = covap.ModelSpec([covap.LayerSpec(f"l{i}", elems) for i in range(16)],
                            bucket_cap_bytes=mb << 20)
    n = 16 * elems
    ng = 3 if n * 4 * 6 < 120e9 else 1
    grads = [torch.empty(n, device="cuda") for _ in range(ng)]
    for i, g in enumerate(grads):
        covap.generate(g, covap.stream_key(1, 0, i))
    out = torch.empty(n, device="cuda")
    for K in (1, 2, 4, 8, 16):
        plan = covap.plan_for(model, covap.CovapConfig(interval=K))
        assert len(plan.buckets) == 16 and len(plan.tensors) == 16
        st = covap.CompressorState(plan, torch.float32, 0)
        cycles = max(1, min(64, int(2e9 // (16 * n * 4)) // K + 1))
        res = {}

        def one(mode, g):
            if mode == "k1f":
                st.filter_unpack(g, out)
            elif mode == "k1":
                st.filter_pack(g, out=out)  # + zero fill of the unselected output
            else:
                st.unpack(out, 1.0, True, selected_only=True)
            st.step_end()

        # Kernel-only time: one K-cycle (every phase once) captured in a CUDA
        # graph and replayed, so the host launch path (Python -> ctypes ->
        # C-ABI, ~10 us per call) cannot starve the GPU at small sizes.
        graph_ms = {}
        cap = torch.cuda.Stream()
        for mode in ("k1f", "k1", "k2"):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap):
                one(mode, grads[0])  # warm-up outside capture (attributes, first launch)
                torch.cuda.synchronize()
                with torch.cuda.graph(gr, stream=cap):
                    for k in range(K):
                        one(mode, grads[k % ng])
            reps = max(3, cycles)
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()  # replay() launches on the current stream
            for _ in range(reps):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            graph_ms[mode] = e0.elapsed_time(e1) / (reps * K)
            del gr
        for mode in ("k1f", "k1", "k2"):
            for _ in range(K):  # warm-up cycle
                st.filter_unpack(grads[0], out) if mode == "k1f" else (
                    st.filter_pack(grads[0], out=out) if mode == "k1" else
                    st.unpack(out, 1.0, True, selected_only=True))
                st.step_end()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            byts = 0
            e0.record()
            for c in range(cycles):
                for k in range(K):
                    _, S = plan.send_elems(st.num_steps)
                    g = grads[(c * K + k) % ng]
                    if mode == "k1f":
                        st.filter_unpack(g, out)
                        byts += 16 * n
                    elif mode == "k1":
                        st.filter_pack(g, out=out)
                        byts += 16 * n
                    else:
                        st.unpack(out, 1.0, True, selected_only=True)
                        byts += 8 * S
                    st.step_end()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / (cycles * K)
            gb = byts / (cycles * K) / 1e9
            res[mode] = (ms, gb / (ms * 1e-3), graph_ms[mode], gb / (graph_ms[mode] * 1e-3))
        rows.append((mb, K, n, res))
        print(mb, K, {k: tuple(round(x, 4) for x in v) for k, v in res.items()}, flush=True)
        del st, plan
    del grads, out
    torch.cuda.empty_cache()
    mb *= 2

lines = ["# Synthetic bucket sweep (BASELINE config 5), one B200\n",
         "16 equal buckets of B MB (N = 16 B / 4 fp32 elements), S = N/K.  Fraction of the "
         f"measured {peak} GB/s copy peak.  K1F = fused single-rank sync (16N bytes); "
         "K1 = filter_pack with the output zero fill (16N); K2 = selected-only unpack (8S); "
         "K1+K2 = the multi-rank kernels together (16N + 8S).  *graph*: one K-cycle "
         "captured in a CUDA graph and replayed (kernel time); *eager*: the same launches "
         "issued one by one from Python through the C-ABI (includes the host launch path, "
         "which dominates below ~8 MB buckets).\n",
         "| bucket | K | N (M elems) | K1F µs graph | K1F frac graph | K1F frac eager | K1 µs graph | "
         "K1 frac graph | K1 frac eager | K2 µs graph | K2 frac graph | K2 frac eager | "
         "K1+K2 frac graph |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for mb, K, n, res in rows:
    c = []
    for m in ("k1f", "k1", "k2"):
        ms, gbs, gms, ggbs = res[m]
        c += [f"{gms * 1e3:.1f}", f"{ggbs / peak:.3f}", f"{gbs / peak:.3f}"]
    (m1, _, g1, gb1), (m2, _, g2, gb2) = res["k1"], res["k2"]
    both = (gb1 * g1 + gb2 * g2) / (g1 + g2)  # bytes over the summed kernel time
    lines.append(f"| {mb} MB | {K} | {n / 1e6:.1f} | " + " | ".join(c) + f" | {both / peak:.3f} |")
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
