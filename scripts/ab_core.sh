#!/bin/bash
# A/B of the core sync kernels: in-tree library vs _variants/$VAR (bench.py lines).
for lib in paper_2311_04499_b200/libcovap_b200.so paper_2311_04499_b200/_variants/${VAR}/libcovap_b200.so; do
  echo "== $lib"
  for rep in 1 2; do
  for cfg in "--layout resnet50 --interval 1" "--layout resnet50 --interval 4" "--layout bert_large --interval 4"; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --no-real-model --steps 30 --warmup 5 2>/dev/null | \
      python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']; u = r.get('unfused_p1', {})
print(d['config']['layout'], d['config']['interval'], 'K1F', r['frac'], 'K1', u.get('k1_frac'), 'K2', u.get('k2_frac'))"
  done; done
done
