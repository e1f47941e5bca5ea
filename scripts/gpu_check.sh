#!/bin/bash
# One GPU session: parity tests, the default bench line, extra workloads, ncu.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
for cfg in "--layout resnet50 --interval 4" "--layout vgg16 --interval 4" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --steps 12 --warmup 4 >> gpurun_out/bench_extra.json 2>> gpurun_out/bench.err
done
cat gpurun_out/bench_extra.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"filter_pack|unpack" -s 4 -c 4 -o gpurun_out/prof_r50 python bench.py --steps 3 --warmup 3 --no-overhead --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_full.log
