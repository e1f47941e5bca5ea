#!/bin/bash
# A/B of the whole-step peer kernel shape: in-tree library vs _variants/* (virtual ranks, one GPU).
for lib in paper_2311_04499_b200/libcovap_b200.so $(ls -d paper_2311_04499_b200/_variants/*/libcovap_b200.so); do
  echo "== $lib"
  COVAP_LIB_PATH=$PWD/$lib timeout 200 python scripts/peer_bench.py --ranks 1,2 --layouts resnet50,bert_large --intervals 1 2>&1 | \
    python -c "import sys,json; [print(d['layout'], d['K'], d['P_virtual'], 'mode1', d['mode1_ms'], 'mode2', d['mode2_ms']) for d in map(json.loads, sys.stdin)]"
done
