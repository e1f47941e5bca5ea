#!/bin/bash
# A/B of top-k kernel variants: in-tree library vs _variants/<NAMES> (bench_baselines top-k).
cd "$(dirname "$0")/.."
for name in ${NAMES:-topk_old topk_segmax topk_segmax_b4}; do
  lib=paper_2311_04499_b200/_variants/$name/libcovap_b200.so
  echo "== $name"
  for L in resnet50 vgg16 bert_large; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout $L --schemes topk --cpu-steps 0 --steps 40 | \
      python -c "import sys,json; [print('$name', d['layout'], d['scheme'], d['ms_per_step'], d.get('roofline_frac')) for d in map(json.loads, sys.stdin)]"
  done
done
