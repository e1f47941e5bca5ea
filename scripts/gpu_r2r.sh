#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r2r}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -3 $O/pytest_fb.log
for L in resnet50 bert_large; do
  timeout 120 python scripts/kernel_timeline.py --layout $L --scheme randomk --steps 3 > $O/timeline_${L}_randomk.txt 2>&1
done
bash scripts/ab_rk.sh | tee $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes randomk --cpu-steps 0 --steps 3 --warmup 2 > /dev/null 2>&1
echo "ncu rc=$?"
