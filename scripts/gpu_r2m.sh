#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2m; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "symmetric" > $O/pytest_sym.log 2>&1
echo "pytest sym rc=$?" >> $O/rc.txt
COVAP_LIB_PATH=$PWD/paper_2311_04499_b200/_variants/evf/libcovap_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fp32_full or zero_filling or fused_single" > $O/pytest_evf.log 2>&1
echo "pytest evf rc=$?" >> $O/rc.txt
NAMES="base evf base evf" timeout 2400 bash scripts/variants.sh run > $O/variants.txt 2> $O/variants.err
echo "variants rc=$?" >> $O/rc.txt
