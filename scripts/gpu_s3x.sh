#!/bin/bash
# K1 (multi-rank, K=1) vs K1F at ResNet-50: ncu full of one launch each.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3x}; mkdir -p $O
timeout 300 ncu --set full --clock-control none -k regex:"filter_kernel" -s 3 -c 1 -o $O/k1f_r50_k1 python scripts/profile_step.py --layout resnet50 --interval 1 --mode fused --iters 5 > /dev/null 2>&1; echo "a rc=$?"
timeout 300 ncu --set full --clock-control none -k regex:"filter_kernel" -s 3 -c 1 -o $O/k1_r50_k1 python scripts/profile_step.py --layout resnet50 --interval 1 --mode unfused --iters 5 > /dev/null 2>&1; echo "b rc=$?"
timeout 300 ncu --set full --clock-control none -k regex:"filter_kernel" -s 3 -c 1 -o $O/k1_r50_k4 python scripts/profile_step.py --layout resnet50 --interval 4 --mode unfused --iters 5 > /dev/null 2>&1; echo "c rc=$?"
