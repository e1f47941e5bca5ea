#!/bin/bash
# ncu captures (launch list + full sets) and extra bench lines for profiles/r2_*.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; rm -f gpurun_out/prof_*.ncu-rep gpurun_out/launches.csv gpurun_out/bench_extra.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" > gpurun_out/r2e_rc.txt
for cfg in "--interval auto" "--layout resnet50 --interval 1" "--layout vgg16 --interval 4" "--layout vgg16 --interval 2" "--layout vgg16 --interval 8" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 400 python bench.py $cfg --no-cpu-baseline --no-overhead --steps 20 --warmup 4 >> gpurun_out/bench_extra.json 2>> gpurun_out/bench.err
done
echo "extra done" >> gpurun_out/r2e_rc.txt
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead > /dev/null 2>&1; echo "ncu launches rc=$?" >> gpurun_out/r2e_rc.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 4 -c 2 -o gpurun_out/prof_r50_k4_fused python scripts/profile_step.py --layout resnet50 --interval 4 --mode fused --iters 6 > gpurun_out/ncu_a.log 2>&1; echo "ncu a rc=$?" >> gpurun_out/r2e_rc.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 8 -c 4 -o gpurun_out/prof_r50_k4_unfused python scripts/profile_step.py --layout resnet50 --interval 4 --mode unfused --iters 6 > gpurun_out/ncu_b.log 2>&1; echo "ncu b rc=$?" >> gpurun_out/r2e_rc.txt
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"filter|unpack" -s 4 -c 2 -o gpurun_out/prof_bert_k4_unfused python scripts/profile_step.py --layout bert_large --interval 4 --mode unfused --iters 3 > gpurun_out/ncu_c.log 2>&1; echo "ncu c rc=$?" >> gpurun_out/r2e_rc.txt
