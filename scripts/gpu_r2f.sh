#!/bin/bash
# compute-sanitizer on the round-2 kernels + real-model timelines of the side-stream schedule.
cd "$(dirname "$0")/.."
O=gpurun_out/r2f; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "selected_unpack or (zero_filling and tablev) or (zero_filling and resnet50-8) or back_to_back or edge_cases or allreduce_mean_rows" > $O/memcheck_split.log 2>&1
echo "memcheck rc=$?" > $O/rc.txt
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "selected_unpack or (zero_filling and tablev)" > $O/racecheck_split.log 2>&1
echo "racecheck rc=$?" >> $O/rc.txt
timeout 600 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "selected_unpack and 1001-77" > $O/synccheck_split.log 2>&1
echo "synccheck rc=$?" >> $O/rc.txt
timeout 1500 python scripts/real_models.py --models resnet50,vgg16,bert_large --intervals 1,4 --trace $O/traces > $O/real_models.jsonl 2> $O/real_models.err
echo "real rc=$?" >> $O/rc.txt
