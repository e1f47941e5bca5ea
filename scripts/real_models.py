"""Real-model DDP steps under the COVAP communication hook (SURVEY.md §8(f)
rank 1) for the three BASELINE model families, one GPU.

For each model: random-init weights, synthetic inputs of the stated shape,
bf16 autocast, fp32 gradients, SGD (momentum 0.9), DDP with 25 MB buckets and
gradient_as_bucket_view.  Modes: the default allreduce-mean hook ("dense") and
the COVAP hook (paper_2311_04499_b200.ddp.CovapDDPHook) at each requested K.
Device time per step (CUDA events around N back-to-back steps).  One JSON
line per model.

    python scripts/real_models.py --models resnet50,vgg16,bert_large --intervals 1,4
"""
import argparse
import json
import os
import socket
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def build(name, dev):
    import torch
    if name == "resnet50":
        import torchvision
        net = torchvision.models.resnet50().to(dev).to(memory_format=torch.channels_last)
        x = torch.randn(64, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (64,), device=dev)
        return net, lambda m: torch.nn.functional.cross_entropy(m(x), y), \
            "torchvision resnet50, batch 64, 224x224"
    if name == "vgg16":
        import torchvision
        net = torchvision.models.vgg16().to(dev).to(memory_format=torch.channels_last)
        x = torch.randn(32, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (32,), device=dev)
        return net, lambda m: torch.nn.functional.cross_entropy(m(x), y), \
            "torchvision vgg16, batch 32, 224x224"
    if name == "bert_large":
        from transformers import BertConfig, BertModel
        cfg = BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                         intermediate_size=4096, vocab_size=30522)
        net = BertModel(cfg).to(dev)
        ids = torch.randint(0, cfg.vocab_size, (16, 128), device=dev)
        tt = torch.zeros_like(ids)

        def loss(m):
            o = m(input_ids=ids, token_type_ids=tt)
            return o.last_hidden_state.float().pow(2).mean() + o.pooler_output.float().mean()
        return net, loss, "HF BertModel (24x1024, vocab 30522), batch 16, seq 128"
    raise ValueError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="resnet50,vgg16,bert_large")
    ap.add_argument("--intervals", default="1,4")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--trace", default="",
                    help="directory: for each COVAP mode also record one step's per-bucket "
                         "timeline (CUDA events, paper_2311_04499_b200.trace) -> Chrome trace")
    ap.add_argument("--free-sms", type=int, default=0,
                    help="side schedule: SMs K1 / K2 leave to the collective / backward")
    ap.add_argument("--schedules", default="fused,side",
                    help="COVAP hook schedules at one rank: 'fused' (K1F on the producing stream) "
                         "and/or 'side' (the multi-rank schedule through a 1-rank NCCL "
                         "communicator: K1 on the producing stream, allreduce + K2 on the side "
                         "stream)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    import paper_2311_04499_b200 as covap
    from paper_2311_04499_b200.ddp import CovapDDPHook

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    sk.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    torch.backends.cudnn.benchmark = True
    scheds = args.schedules.split(",")
    modes = ["dense"] + [(int(k), sc) for k in args.intervals.split(",") for sc in scheds]
    comm1 = covap.Communicator(covap.Communicator.unique_id(), 1, 0, 0) if "side" in scheds else None
    for name in args.models.split(","):
        res, info = {}, {}
        for mode in modes:
            torch.manual_seed(0)
            net, loss_fn, desc = build(name, dev)
            model = DDP(net, device_ids=[0], bucket_cap_mb=25, gradient_as_bucket_view=True)
            hook = None
            if mode != "dense":
                k, sc = mode
                hook = CovapDDPHook(covap.CovapConfig(interval=k), comm1 if sc == "side" else None,
                                    0, warmup=2, fuse_single_rank=sc == "fused",
                                    free_sms=args.free_sms)
                model.register_comm_hook(hook, CovapDDPHook.hook)
            opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)

            def step():
                with torch.autocast("cuda", dtype=torch.bfloat16):
                    loss = loss_fn(model)
                loss.backward()
                opt.step()
                opt.zero_grad(set_to_none=False)

            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                step()
            e1.record()
            torch.cuda.synchronize(dev)
            res[str(mode)] = e0.elapsed_time(e1) / args.steps
            tl_info = None
            if hook is not None and args.trace and hook.sync is not None:
                from paper_2311_04499_b200 import trace
                tl = trace.record_step(hook.sync, step)
                k, sc = mode
                os.makedirs(args.trace, exist_ok=True)
                trace.chrome_trace(os.path.join(args.trace, f"trace_{name}_K{k}_{sc}.json"), tl)
                last = len(tl) - 1
                # what runs after the last bucket's gradient is ready: its K1 and
                # whatever is still on the side stream (collectives, unpacks)
                tail = max(r["k2_end"] for r in tl) - tl[last]["k1_start"]
                tl_info = {"buckets": len(tl),
                           "k1_ms": [round(r["k1_end"] - r["k1_start"], 4) for r in tl],
                           "side_ms": [round(r["k2_end"] - r["comm_start"], 4)
                                       if r["comm_start"] >= 0 else None for r in tl],
                           "sync_after_last_gradient_ms": round(tail, 4),
                           "sync_after_last_gradient_frac_of_step": round(tail / res[str(mode)], 5)}
            if hook is not None:
                info[str(mode)] = {"timeline": tl_info, "hook_active": hook.sync is not None,
                                   "buckets": len(hook.plan.buckets) if hook.plan else None,
                                   "tensors": len(hook.plan.tensors) if hook.plan else None,
                                   "params": sum(b.numel for b in hook.plan.buckets) if hook.plan else None}
            del model, net, opt
            torch.cuda.empty_cache()
        dense = res["dense"]
        line = {"model": name, "desc": desc + ", bf16 autocast, fp32 grads, SGD, DDP 25 MB buckets, 1 GPU",
                "step_ms_dense": round(dense, 3)}
        for k, sc in modes[1:]:
            key = str((k, sc))
            line[f"step_ms_covap_K{k}_{sc}"] = round(res[key], 3)
            line[f"overhead_K{k}_{sc}"] = round((res[key] - dense) / dense, 5)
            line[f"hook_K{k}_{sc}"] = info[key]
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
