#!/bin/bash
# Session 3 evidence: full GPU suite, smoke, default bench line + extra
# workloads, launch list of the bench command.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3t}; mkdir -p $O
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" > $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
for cfg in "--interval auto" "--layout vgg16 --interval 4" "--layout bert_large --interval 4" "--layout bert_large --interval 1"; do
  timeout 300 python bench.py $cfg --no-cpu-baseline --no-overhead --no-real-model >> $O/bench_extra.jsonl 2>> $O/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead --no-real-model > /dev/null 2>&1; echo "ncu rc=$?" >> $O/rc.txt
