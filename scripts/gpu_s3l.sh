#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-s3l}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_feedback.py tests/test_cxx_dropin.py -q -m gpu -x > $O/pytest_fb.log 2>&1; echo "pytest rc=$?" | tee $O/rc.txt
tail -2 $O/pytest_fb.log
for L in resnet50 vgg16 bert_large; do
  timeout 600 python scripts/bench_baselines.py --layout $L --cpu-steps 0 --steps 40 > $O/f4_$L.jsonl 2> $O/f4_$L.err
  python -c "import sys,json; [print(d['layout'], d['scheme'], d['ms_per_step']) for d in map(json.loads, open('$O/f4_$L.jsonl'))]"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/launches_topk_r50.csv \
  python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 3 --warmup 2 > /dev/null 2>&1
timeout 600 ncu -k regex:topk_collect --set full -c 1 --import-source on --clock-control none -o $O/collect_r50 \
  python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 2 --warmup 1 > /dev/null 2>&1
echo "ncu rc=$?"
