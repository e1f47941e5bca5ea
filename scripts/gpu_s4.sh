#!/bin/bash
# Session-4 confirmation pass on a restored container: GPU tests, smoke,
# default bench line, reference arm, launch list.  Output under gpurun_out/s4.
cd "$(dirname "$0")/.."
O=gpurun_out/s4; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/rc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/rc.txt
cat $O/bench.json | head -c 600; echo
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" | tee -a $O/rc.txt
head -c 600 $O/bench_ref.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-overhead > /dev/null 2>&1; echo "ncu rc=$?" | tee -a $O/rc.txt
