#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3i}; mkdir -p $O
SCHEMES=topk bash scripts/ab_rk2.sh > $O/ab_topk.txt 2>&1; sort $O/ab_topk.txt
for lib in paper_2311_04499_b200/libcovap_b200.so paper_2311_04499_b200/_variants/oldcollect/libcovap_b200.so; do
  tag=$(echo $lib | awk -F/ '{print $(NF-1)}')
  COVAP_LIB_PATH=$PWD/$lib timeout 600 ncu -k regex:topk_collect --set full -c 1 --clock-control none -o $O/collect_bert_$tag \
    python scripts/bench_baselines.py --layout bert_large --schemes topk --cpu-steps 0 --steps 2 --warmup 1 > /dev/null 2>&1
  echo "ncu $tag rc=$?"
done
