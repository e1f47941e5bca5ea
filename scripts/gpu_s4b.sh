#!/bin/bash
# Session-4 follow-up: the C++ drop-in GPU cases, extra layouts, baseline compressors.
cd "$(dirname "$0")/.."
O=gpurun_out/s4b; mkdir -p $O
timeout 600 python -m pytest tests/test_cxx_dropin.py -q -m gpu -p no:cacheprovider > $O/pytest_cxx.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_cxx.log
rm -f $O/bench_extra.jsonl
for cfg in "--layout vgg16 --interval 4" "--layout bert_large --interval 4" "--layout resnet50 --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --steps 20 --warmup 4 >> $O/bench_extra.jsonl 2>> $O/bench.err
done
echo "extra rc=$?"
for L in resnet50 vgg16 bert_large; do
  timeout 300 python scripts/bench_baselines.py --layout $L --cpu-steps 0 --steps 40 >> $O/f4.jsonl 2>> $O/f4.err
done
echo "f4 rc=$?"
