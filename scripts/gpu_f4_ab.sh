#!/bin/bash
# A/B of the baseline-compressor kernels: in-tree build vs a variant library.
mkdir -p gpurun_out
for lib in paper_2311_04499_b200/_variants/${VAR:-nopf}/libcovap_b200.so paper_2311_04499_b200/libcovap_b200.so; do
  echo "== $lib"
  for L in resnet50 bert_large; do
    COVAP_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_baselines.py --layout $L --schemes topk,randomk,fp16 --cpu-steps 0 --steps 30 | \
      python -c "import sys,json; [print(d['layout'], d['scheme'], d['ms_per_step'], d['dense_equiv_GBps']) for d in map(json.loads, sys.stdin)]"
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/f4_launches3.csv python scripts/bench_baselines.py --layout resnet50 --schemes topk,randomk,fp16 --steps 2 --warmup 1 --cpu-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/f4_launches3.csv
