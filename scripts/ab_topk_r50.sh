#!/bin/bash
# top-k ResNet-50 (the vector compensation path) A/B over the in-tree lib and _variants/*.
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
for lib in paper_2311_04499_b200/libcovap_b200.so $(ls -d paper_2311_04499_b200/_variants/*/libcovap_b200.so); do
  COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 60 2>/dev/null | \
    python -c "import sys,json; [print('$lib'.split('/')[-2], d['layout'], d['scheme'], d['ms_per_step']) for d in map(json.loads, sys.stdin)]"
done; done
