#!/bin/bash
# Session 3 of round 2: NVLS / NCCL device-API probe, baseline-compressor
# table on HEAD (random-k op 6), launch list of the random-k step.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3b}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
NCCL_DEBUG=WARN timeout 120 ./scripts/nvls_probe > $O/nvls_probe.txt 2>&1; echo "probe rc=$?" >> $O/nvls_probe.txt
for L in resnet50 vgg16 bert_large; do
  timeout 600 python scripts/bench_baselines.py --layout $L --cpu-steps 0 --steps 40 > $O/f4_$L.jsonl 2> $O/f4_$L.err
done
for L in resnet50 bert_large; do
  timeout 120 python scripts/kernel_timeline.py --layout $L --scheme randomk --steps 3 > $O/timeline_${L}_randomk.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_rk_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes randomk --cpu-steps 0 --steps 3 --warmup 2 > /dev/null 2>&1
echo "ncu rc=$?"
