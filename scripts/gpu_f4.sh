#!/bin/bash
# Baseline compressors on one B200: step times, the reference
# CPU arm, and a launch list + full ncu capture of the top-k pass.
mkdir -p gpurun_out
rm -f gpurun_out/f4_bench.jsonl
for L in resnet50 vgg16 bert_large; do
  timeout 600 python scripts/bench_baselines.py --layout $L --k-fraction 0.01 --cpu-steps 1 >> gpurun_out/f4_bench.jsonl 2>> gpurun_out/f4_bench.err
done
cat gpurun_out/f4_bench.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f4_launches.csv \
  python scripts/bench_baselines.py --layout resnet50 --steps 2 --warmup 1 --cpu-steps 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
