#!/bin/bash
# Build kernel design-space variants (here) or run them (on the GPU box).
#   bash scripts/variants.sh build
#   bash scripts/variants.sh run > gpurun_out/variants.txt
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
# Knobs of csrc/covap_kernels.cu: COVAP_K1_TILE / COVAP_K1_STAGES (K1, K1F),
# COVAP_K2_TILE / COVAP_K2_STAGES (K2), COVAP_PDL.  Earlier variants (STG
# outputs, STG zero fill, in-place slots, 2 CTAs/SM) were measured slower and
# removed from the kernels; see profiles/r1_design_study.md.
declare -A V=(
  [base]=""
  [nopdl]="-DCOVAP_PDL=0"
  [k1t16]="-DCOVAP_K1_TILE=16384"
  [k2w1]="-DCOVAP_K2_MIN_WAVES=1"
  [k2w2]="-DCOVAP_K2_MIN_WAVES=2"
  [k2w4]="-DCOVAP_K2_MIN_WAVES=4"
  [k12w2]="-DCOVAP_K1_MIN_WAVES=2 -DCOVAP_K2_MIN_WAVES=2"
  [k2t16]="-DCOVAP_K2_TILE=16384 -DCOVAP_K2_STAGES=6"
  [evf]="-DCOVAP_EVICT_FIRST=1"
)
if [ "$1" = "build" ]; then
  for name in "${!V[@]}"; do
    out=$ROOT/paper_2311_04499_b200/_variants/$name
    mkdir -p $out
    make -s -C $ROOT/paper_2311_04499_b200/csrc OUT=$out/libcovap_b200.so OBJ=$out/obj KDEFS="${V[$name]}"
  done
  exit 0
fi
if [ "$1" = "k12" ]; then  # graph-timed K1 / K2 of the multi-rank step per variant
  for name in ${NAMES:-base k2w1 k2w2 k2w4 k12w2 k2t16}; do
    lib=$ROOT/paper_2311_04499_b200/_variants/$name/libcovap_b200.so
    COVAP_LIB_PATH=$lib timeout 600 python $ROOT/scripts/k12_graph.py --label $name \
      --layouts resnet50:4,resnet50:1,vgg16:4,bert_large:4 2>/dev/null
  done
  exit 0
fi
for name in ${NAMES:-base evf}; do
  lib=$ROOT/paper_2311_04499_b200/_variants/$name/libcovap_b200.so
  for cfg in "--layout resnet50 --interval 4" "--layout resnet50 --interval 1" "--layout vgg16 --interval 4" "--layout bert_large --interval 4"; do
    COVAP_LIB_PATH=$lib timeout 300 python $ROOT/bench.py $cfg --no-cpu-baseline --no-overhead --steps 30 --warmup 5 2>/dev/null | \
      python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']; u = r.get('unfused_p1', {}).get('graph', {})
print('$name', d['config']['layout'], 'K%d' % d['details']['interval'], 'value %.0f' % d['value'],
      'k1f %.3f' % r['frac'], 'k1 %.3f' % u.get('k1_frac', 0), 'k2 %.3f' % u.get('k2_frac', 0),
      'e2e %.1f' % d['e2e']['value'])"
  done
done
