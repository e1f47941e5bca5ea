#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2j; mkdir -p $O
for name in topk_vmask topk_vmask_d4; do
  COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/$name/libcovap_b200.so timeout 900 python -m pytest tests/test_gpu_feedback.py -q -p no:cacheprovider -k "topk or Topk" > $O/pytest_$name.log 2>&1
  echo "pytest $name rc=$?" >> $O/rc.txt
done
NAMES="topk_old topk_vmax topk_vmask topk_vmask_u16 topk_vmask_d4 topk_vmax_d4" timeout 1500 bash scripts/ab_topk.sh > $O/ab_topk.txt 2> $O/ab_topk.err
echo "ab rc=$?" >> $O/rc.txt
for name in topk_vmask topk_vmask_d4; do
  COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/$name/libcovap_b200.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/topk_$name.csv -k regex:"collect" python scripts/bench_baselines.py --layout resnet50 --schemes topk --cpu-steps 0 --steps 6 > $O/topk_$name.out 2>&1
done
