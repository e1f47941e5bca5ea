#!/bin/bash
# compute-sanitizer over session 3's kernels: the compacting top-k collect,
# the vector / work-unit compensation pass, the NCCL-window peer kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3u}; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
K='edge_cases or (full_layout and topk and resnet50) or (virtual_rank and topk)'
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x -k "$K" > $O/memcheck_fb.log 2>&1; echo "memcheck fb rc=$?" | tee -a $O/rc.txt
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x -k "edge_cases and topk" > $O/racecheck_fb.log 2>&1; echo "racecheck fb rc=$?" | tee -a $O/rc.txt
timeout 1200 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_multiproc.py -q -m gpu -x -k "nccl_window and P1" > $O/memcheck_peer.log 2>&1; echo "memcheck peer rc=$?" | tee -a $O/rc.txt
for f in $O/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -4; done
