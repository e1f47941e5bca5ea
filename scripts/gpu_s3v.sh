#!/bin/bash
# random-k tail-tile fix: the new wire test on the previous build (expected
# to fail) and on the fix; sanitizers over the session's kernels; C++ API.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3v}; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/old/libcovap_b200.so timeout 600 python -m pytest tests/test_gpu_feedback.py -q -m gpu -k "virtual_rank and tail-tensor" > $O/old_tail.log 2>&1; echo "old lib tail-tensor rc=$?" | tee -a $O/rc.txt
tail -3 $O/old_tail.log
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu > $O/fb.log 2>&1; echo "fixed feedback suite rc=$?" | tee -a $O/rc.txt
tail -2 $O/fb.log
K='edge_cases or (full_layout and resnet50) or (virtual_rank and tail-tensor and 2-)'
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_feedback.py -q -m gpu -k "$K" > $O/memcheck_fb.log 2>&1; echo "memcheck fb rc=$?" | tee -a $O/rc.txt
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_feedback.py -q -m gpu -k "edge_cases and ints" > $O/racecheck_fb.log 2>&1; echo "racecheck fb rc=$?" | tee -a $O/rc.txt
timeout 900 python -m pytest tests/test_cxx_dropin.py -q -m gpu > $O/cxx.log 2>&1; echo "cxx rc=$?" | tee -a $O/rc.txt
tail -2 $O/cxx.log
for f in $O/memcheck_fb.log $O/racecheck_fb.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -4; done
