#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2h; mkdir -p $O
for name in topk_old topk_segmax_b4; do
  COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/$name/libcovap_b200.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/topk_$name.csv -k regex:"compensate|topk" python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 6 > $O/topk_$name.out 2>&1
  echo "$name rc=$?" >> $O/rc.txt
done
