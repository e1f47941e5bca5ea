#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2g; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_feedback.py tests/test_cxx_dropin.py -q -p no:cacheprovider > $O/pytest_feedback.log 2>&1
echo "pytest rc=$?" > $O/rc.txt
timeout 1500 bash scripts/ab_topk.sh > $O/ab_topk.txt 2> $O/ab_topk.err
echo "ab rc=$?" >> $O/rc.txt
