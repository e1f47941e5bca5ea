"""Peer-collective modes on ONE GPU with P virtual ranks (not an NVLink
measurement: peer loads are local HBM loads here, and the ranks share the
GPU's 148 SMs).  Shows what the one-kernel step (mode 2) costs against the
K1 kernel + collective kernel pair (modes 0/1) when the exchange itself is
nearly free, i.e. the fixed cost of each schedule.

    python scripts/peer_bench.py --layouts resnet50,bert_large --intervals 1,4 --ranks 1,2,4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layouts", default="resnet50,bert_large")
    ap.add_argument("--intervals", default="1,4")
    ap.add_argument("--ranks", default="1,2,4")
    ap.add_argument("--steps", type=int, default=12)
    a = ap.parse_args()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for name in a.layouts.split(","):
        for K in map(int, a.intervals.split(",")):
            plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
            d = plan.total_numel()
            for P in map(int, a.ranks.split(",")):
                if name == "bert_large" and P > 2:
                    continue  # memory: P x (g, r, out, 2 send buffers) of 1.34 GB
                states = [covap.CompressorState(plan, torch.float32, 0) for _ in range(P)]
                groups = [covap.PeerGroup(st, P, r) for r, st in enumerate(states)]
                covap.PeerGroup.attach_local(groups)
                streams = [torch.cuda.Stream() for _ in range(P)]
                grads = []
                for r in range(P):
                    g = torch.empty(d, device="cuda")
                    covap.generate(g, covap.stream_key(1, r, 0))
                    grads.append(g)
                outs = [torch.empty(d, device="cuda") for _ in range(P)]
                line = {"layout": name, "K": K, "P_virtual": P, "elements": d}
                for mode in (1, 2):
                    for g in groups:
                        g.set_limits(max_ctas=max(1, sms // P) if mode == 2 else max(1, sms // (2 * P)),
                                     timeout_s=10.0)
                        g.set_fused(mode)

                    def step():
                        main = torch.cuda.current_stream()
                        for r in range(P):
                            streams[r].wait_stream(main)
                            groups[r].sync(grads[r], outs[r], streams[r])
                        for r in range(P):
                            main.wait_stream(streams[r])

                    for _ in range(3):
                        step()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.steps):
                        step()
                    e1.record()
                    torch.cuda.synchronize()
                    for g in groups:
                        g.check()
                    line[f"mode{mode}_ms"] = round(e0.elapsed_time(e1) / a.steps, 4)
                print(json.dumps(line), flush=True)
                del states, groups, grads, outs
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
