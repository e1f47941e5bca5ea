#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3h}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -2 $O/pytest_fb.log
SCHEMES=topk bash scripts/ab_rk2.sh > $O/ab_topk.txt 2>&1; sort $O/ab_topk.txt
for L in resnet50 bert_large; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/launches_topk_$L.csv \
  python scripts/bench_baselines.py --layout $L --schemes topk --cpu-steps 0 --steps 2 --warmup 1 > /dev/null 2>&1
done
echo "ncu rc=$?"
