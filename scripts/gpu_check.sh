#!/bin/bash
# One GPU session: parity tests, the default bench line, extra workloads, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
rm -f gpurun_out/bench_extra.json
for cfg in "--layout resnet50 --interval 4" "--layout vgg16 --interval 4" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --steps 12 --warmup 4 >> gpurun_out/bench_extra.json 2>> gpurun_out/bench.err
done
cat gpurun_out/bench_extra.json
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead > /dev/null 2>&1; echo "ncu1 rc=$?"
for m in fused unfused; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 2 -c 4 -o gpurun_out/prof_r50_k1_$m python scripts/profile_step.py --layout resnet50 --interval 1 --mode $m --iters 4 > gpurun_out/ncu_$m.log 2>&1; echo "ncu $m rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 2 -c 4 -o gpurun_out/prof_r50_k4_unfused python scripts/profile_step.py --layout resnet50 --interval 4 --mode unfused --iters 4 > gpurun_out/ncu_k4.log 2>&1; echo "ncu k4 rc=$?"
fi
