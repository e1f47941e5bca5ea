#!/bin/bash
# broader memcheck: the whole baseline-compressor suite, the peer kernels
# (virtual ranks, modes 0/1/2), the host pipeline and DDP hook.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3w}; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_feedback.py -q -m gpu > $O/memcheck_fb_all.log 2>&1; echo "memcheck feedback rc=$?" | tee -a $O/rc.txt
timeout 2400 $CS --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "peer or host or fused_sgd or symmetric" > $O/memcheck_parity.log 2>&1; echo "memcheck parity rc=$?" | tee -a $O/rc.txt
for f in $O/memcheck_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed" $f | tail -3; done
