#!/bin/bash
# random-k collision-free fast path: feedback suite, memcheck of the new
# kernels, A/B vs the previous selection (hash / sort + free SMs).
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3rk}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/fb.log 2>&1; echo "feedback rc=$?" | tee -a $O/rc.txt
tail -2 $O/fb.log
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x -k "edge_cases or (virtual_rank and tail-tensor and 2-) or (full_layout and resnet50)" > $O/memcheck.log 2>&1; echo "memcheck rc=$?" | tee -a $O/rc.txt
grep -E "ERROR SUMMARY|passed|failed" $O/memcheck.log | tail -2
SCHEMES=randomk bash scripts/ab_rk2.sh 2>&1 | sort | tee $O/ab.txt
