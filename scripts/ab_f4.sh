#!/bin/bash
# A/B of baseline-compressor variants: in-tree library vs _variants/* (bench_baselines, $SCHEMES).
for lib in paper_2311_04499_b200/libcovap_b200.so $(ls -d paper_2311_04499_b200/_variants/*/libcovap_b200.so); do
  echo "== $lib"
  for L in resnet50 bert_large; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout $L --schemes ${SCHEMES:-fp16} --cpu-steps 0 --steps 40 | \
      python -c "import sys,json; [print(d['layout'], d['scheme'], d['ms_per_step']) for d in map(json.loads, sys.stdin)]"
  done
done
