"""Host-buffer sync step (covap_sync_step_host) back to back, per chunk size
and staging aliasing (probe, not product): GB/s = 4N / step time."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2311_04499_b200 as covap  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for name in os.environ.get("LAYOUTS", "resnet50,bert_large").split(","):
        plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=4))
        n = plan.total_numel()
        hin = [torch.empty(n, pin_memory=True) for _ in range(2)]
        hout = torch.empty(n, pin_memory=True)
        dg, do = torch.empty(n, device=dev), torch.empty(n, device=dev)
        for chunk in [int(x) for x in os.environ.get("CHUNKS", "0,2097152,8388608,16777216").split(",")]:
            for alias in (True, False):
                sync = covap.CovapSync(plan, None, torch.float32, 0)
                out = dg if alias else do
                for s in range(3):
                    sync.sync_host(hin[s % 2], hout, dg, out, chunk, stream)
                torch.cuda.synchronize()
                steps = 10
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for s in range(steps):
                    sync.sync_host(hin[s % 2], hout, dg, out, chunk, stream)
                b.record(stream)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / steps
                print(json.dumps({"layout": name, "chunk": chunk, "alias": alias,
                                  "ms": round(ms, 4), "gbs": round(4 * n / ms / 1e6, 2)}),
                      flush=True)
                del sync


if __name__ == "__main__":
    main()
