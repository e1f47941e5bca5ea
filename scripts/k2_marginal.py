"""K2's cost inside the multi-rank step sequence (probe, not product).

The bench's `unfused_p1.graph.k2_ms` replays K2 launches back to back, so a
K2's ramp overlaps the previous K2's tail (programmatic dependent launch).
In a real step K2 follows K1 -> allreduce.  Measured here, per layout and K,
one K-cycle captured in a CUDA graph each (1-rank NCCL communicator):

  k1c1     [K1, C1] per step
  k1c1k2   [K1, C1, K2] per step          -> K2 marginal = k1c1k2 - k1c1
  k2       [K2] per step (the bench's graph number)
  eager    K1, C1, K2 issued from Python behind a 500 us head-start spin,
           events around K2
"""
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
    comm = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0)
    for name, K in (("resnet50", 4), ("resnet50", 1), ("vgg16", 4), ("bert_large", 4)):
        plan = covap.plan_for(covap.load_layout(name), covap.CovapConfig(interval=K))
        sync = covap.CovapSync(plan, comm, torch.float32, 0, fuse_single_rank=False)
        st = sync.state
        n = plan.total_numel()
        grads = [torch.empty(n, device=dev) for _ in range(3)]
        for i, g in enumerate(grads):
            covap.generate(g, covap.stream_key(1, 0, i))
        out = torch.empty(n, device=dev)

        def k1(k):
            st.num_steps = k
            st.filter_pack(grads[k % 3], out=out)

        def c1(k):
            se, _ = plan.send_elems(k)
            if se:
                comm.allreduce(st.send[:se])

        def k2(k):
            st.num_steps = k
            st.unpack(out, 1.0, True, selected_only=True)

        def cycle(fns):
            cap = torch.cuda.Stream(dev)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap):
                for f in fns:
                    f(0)
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(gr, stream=cap):
                    for k in range(K):
                        for f in fns:
                            f(k)
            gr.replay()
            torch.cuda.synchronize(dev)
            reps = 20
            a, b = ev(), ev()
            a.record(stream)
            for _ in range(reps):
                gr.replay()
            b.record(stream)
            torch.cuda.synchronize(dev)
            return a.elapsed_time(b) / (reps * K) * 1e3  # us per step

        def sync_step(k):  # the public multi-rank call (covap_sync_step)
            if k == 0:
                st.num_steps = 0
            sync.sync(grads[k % 3], out)

        t_sync = cycle([sync_step])
        t_k1c1 = cycle([k1, c1])
        t_all = cycle([k1, c1, k2])
        t_k2 = cycle([k2])
        # eager with a head start
        eg = []
        for i in range(3 * K):
            k = i % K
            covap.spin(500.0, 1, stream)
            k1(k)
            c1(k)
            a, b = ev(), ev()
            a.record(stream)
            k2(k)
            b.record(stream)
            eg.append((a, b))
        torch.cuda.synchronize(dev)
        t_eager = sum(a.elapsed_time(b) for a, b in eg[K:]) / (2 * K) * 1e3
        S = sum(plan.send_elems(k)[1] for k in range(K)) / K
        k2b = 8 * S
        print(json.dumps({
            "layout": name, "K": K, "n": n, "S_avg": S,
            "sync_step_us": round(t_sync, 2),
            "sync_step_frac": round((16 * n + k2b) / (t_sync * 1e-6) / 1e9 / PEAK, 4),
            "k1c1_us": round(t_k1c1, 2), "k1c1k2_us": round(t_all, 2),
            "k2_marginal_us": round(t_all - t_k1c1, 2), "k2_graph_us": round(t_k2, 2),
            "k2_eager_us": round(t_eager, 2),
            "k2_frac_marginal": round(k2b / ((t_all - t_k1c1) * 1e-6) / 1e9 / PEAK, 4),
            "k2_frac_graph": round(k2b / (t_k2 * 1e-6) / 1e9 / PEAK, 4),
            "k2_frac_eager": round(k2b / (t_eager * 1e-6) / 1e9 / PEAK, 4),
            "step_frac": round((16 * n + k2b) / (t_all * 1e-6) / 1e9 / PEAK, 4),
        }), flush=True)
        del sync, st, grads, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
