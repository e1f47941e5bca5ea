#!/bin/bash
# random-k merged selection chain: feedback tests, f4 numbers, timeline, launches.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3c}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -3 $O/pytest_fb.log
for L in resnet50 vgg16 bert_large; do
  timeout 600 python scripts/bench_baselines.py --layout $L --schemes randomk --cpu-steps 0 --steps 40 > $O/rk_$L.jsonl 2> $O/rk_$L.err
  cut -c1-200 $O/rk_$L.jsonl
done
for L in resnet50 bert_large; do
  timeout 120 python scripts/kernel_timeline.py --layout $L --scheme randomk --steps 3 > $O/timeline_${L}_randomk.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_rk_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes randomk --cpu-steps 0 --steps 3 --warmup 2 > /dev/null 2>&1
echo "ncu rc=$?"
