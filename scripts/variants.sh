#!/bin/bash
# Build kernel design-space variants (here) or run them (on the GPU box).
#   bash scripts/variants.sh build
#   bash scripts/variants.sh run > gpurun_out/variants.txt
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
declare -A V=(
  [pdl]=""
  [nopdl]="-DCOVAP_PDL=0"
)
if [ "$1" = "build" ]; then
  for name in "${!V[@]}"; do
    out=$ROOT/paper_2311_04499_b200/_variants/$name
    mkdir -p $out
    make -s -C $ROOT/paper_2311_04499_b200/csrc OUT=$out/libcovap_b200.so OBJ=$out/obj KDEFS="${V[$name]}"
  done
  exit 0
fi
for name in ${NAMES:-pdl nopdl}; do
  lib=$ROOT/paper_2311_04499_b200/_variants/$name/libcovap_b200.so
  for cfg in "--layout resnet50 --interval 1" "--layout resnet50 --interval 4" "--layout vgg16 --interval 4" "--layout bert_large --interval 1" "--layout bert_large --interval 4"; do
    COVAP_LIB_PATH=$lib timeout 300 python $ROOT/bench.py $cfg --no-cpu-baseline --no-overhead --steps 30 --warmup 5 2>/dev/null | \
      python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']; u = r.get('unfused_p1', {})
print('$name', d['config']['layout'], 'K%d' % d['config']['interval'], 'value %.0f' % d['value'],
      'k1f %.3f' % r['frac'], 'k1 %.3f' % u.get('k1_frac', 0), 'k2 %.3f' % u.get('k2_frac', 0))"
  done
done
