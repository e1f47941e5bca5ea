#!/bin/bash
# One GPU session: parity tests, the default bench line, extra workloads, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
rm -f gpurun_out/bench_extra.json
for cfg in "--layout resnet50 --interval 4" "--layout vgg16 --interval 4" "--layout vgg16 --interval 2" "--layout vgg16 --interval 8" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --steps 20 --warmup 4 >> gpurun_out/bench_extra.json 2>> gpurun_out/bench.err
done
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 2 -c 2 -o gpurun_out/prof_r50_k1_fused python scripts/profile_step.py --layout resnet50 --interval 1 --mode fused --iters 4 > gpurun_out/ncu_a.log 2>&1; echo "ncu a rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 4 -c 4 -o gpurun_out/prof_r50_k4_unfused python scripts/profile_step.py --layout resnet50 --interval 4 --mode unfused --iters 4 > gpurun_out/ncu_b.log 2>&1; echo "ncu b rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 1 -c 1 -o gpurun_out/prof_bert_k1_fused python scripts/profile_step.py --layout bert_large --interval 1 --mode fused --iters 2 > gpurun_out/ncu_c.log 2>&1; echo "ncu c rc=$?"
fi
