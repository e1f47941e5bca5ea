#!/bin/bash
# Sparsifier rework check: feedback GPU tests, A/B of top-k / random-k step
# times (HEAD~ library vs new), kernel timelines, ncu launch list.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r2n}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -3 $O/pytest_fb.log
for L in resnet50 bert_large; do for S in topk randomk; do
  timeout 120 python scripts/kernel_timeline.py --layout $L --scheme $S --steps 3 > $O/timeline_${L}_$S.txt 2>&1
done; done
for rep in 1 2; do
for lib in paper_2311_04499_b200/_variants/old/libcovap_b200.so paper_2311_04499_b200/libcovap_b200.so; do
  for L in resnet50 vgg16 bert_large; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout $L --schemes ${SCHEMES:-topk,randomk} --cpu-steps 0 --steps 40 2>>$O/ab.err | \
      python -c "import sys,json; [print('$lib'.split('/')[-2], d['layout'], d['scheme'], d['ms_per_step']) for d in map(json.loads, sys.stdin)]"
  done
done
done | tee $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes topk,randomk --cpu-steps 0 --steps 3 --warmup 2 > /dev/null 2>&1
echo "ncu rc=$?"
