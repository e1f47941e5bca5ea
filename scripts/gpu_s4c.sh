#!/bin/bash
# Session-4 ncu: the headline kernel (K1F, ResNet-50 K=4) and K1 / K2 of the multi-rank step, fresh build.
cd "$(dirname "$0")/.."
O=gpurun_out/s4c; mkdir -p $O
timeout 300 python scripts/profile_step.py --layout resnet50 --interval 4 --mode fused --iters 4 > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 4 -c 4 -o $O/r50_k4_fused python scripts/profile_step.py --layout resnet50 --interval 4 --mode fused --iters 4 > $O/ncu_a.log 2>&1; echo "ncu a rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 4 -c 4 -o $O/r50_k4_unfused python scripts/profile_step.py --layout resnet50 --interval 4 --mode unfused --iters 4 > $O/ncu_b.log 2>&1; echo "ncu b rc=$?"
