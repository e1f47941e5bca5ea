#!/bin/bash
# A/B of baseline-compressor kernel variants (paper_2311_04499_b200/_variants/*).
for lib in paper_2311_04499_b200/libcovap_b200.so $(ls -d paper_2311_04499_b200/_variants/*/libcovap_b200.so); do
  echo "== $lib"
  for L in resnet50 vgg16 bert_large; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout $L --schemes ${SCHEMES:-topk} --cpu-steps 0 --steps 30 | \
      python -c "import sys,json; [print(d['layout'], d['scheme'], d['ms_per_step'], d['dense_equiv_GBps']) for d in map(json.loads, sys.stdin)]"
  done
done
