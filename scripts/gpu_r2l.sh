#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2l; mkdir -p $O
COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/k2s64/libcovap_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "selected_unpack or zero_filling or overlapped or multi_rank_code or peer_collective_fp32 or back_to_back or host_pipeline" > $O/pytest_k2s64.log 2>&1
echo "pytest k2s64 rc=$?" >> $O/rc.txt
NAMES="base k2s4 k2s16 k2s64" timeout 1500 bash scripts/variants.sh k12 > $O/k12_variants.jsonl 2> $O/k12.err
echo "k12 rc=$?" >> $O/rc.txt
for name in base k2s16; do
  COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/$name/libcovap_b200.so timeout 600 python scripts/sweep.py --max-mb 16 --out $O/sweep_$name.md > $O/sweep_$name.log 2>&1
  echo "sweep $name rc=$?" >> $O/rc.txt
done
