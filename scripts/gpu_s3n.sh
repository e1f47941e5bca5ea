#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3n}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -2 $O/pytest_fb.log
SCHEMES=${SCHEMES:-topk} bash scripts/ab_rk2.sh 2>&1 | sort > $O/ab.txt; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/launches_topk_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 2 --warmup 1 > /dev/null 2>&1
echo "ncu rc=$?"
