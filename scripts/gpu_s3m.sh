#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3m}; mkdir -p $O
SCHEMES=topk bash scripts/ab_rk2.sh 2>&1 | sort > $O/ab_topk.txt; cat $O/ab_topk.txt
timeout 600 ncu -k regex:compensate_kernel --set full -c 1 --import-source on --clock-control none -o $O/compensate_r50 \
  python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 2 --warmup 1 > /dev/null 2>&1
echo "ncu rc=$?"
timeout 300 python bench.py --no-real-model > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench.json'));print(d['ms_per_step'], d['roofline']['frac'])"
