#!/bin/bash
# Round-2 first GPU pass: multi-process IPC tests, new parity tests, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi -L > $O/env.txt 2>&1; which nvidia-cuda-mps-control >> $O/env.txt 2>&1
nproc >> $O/env.txt; free -g >> $O/env.txt
timeout 900 python -m pytest tests/test_multiproc.py -x -q -k "resnet50-K4-P2-mode1" > $O/mp_first.log 2>&1
echo "first rc=$?" >> $O/env.txt
timeout 1800 python -m pytest tests/test_multiproc.py -q > $O/mp_all.log 2>&1
echo "mp rc=$?" >> $O/env.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "allreduce_mean or normwise or back_to_back" > $O/parity_new.log 2>&1
echo "parity rc=$?" >> $O/env.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/env.txt
