#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2c; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "allreduce_mean or back_to_back or zero_filling or K8-P2-mode0 or ddp_hook" > $O/pytest_fix.log 2>&1
echo "pytest rc=$?" > $O/rc.txt
timeout 1800 bash scripts/variants.sh k12 > $O/k12_variants.jsonl 2> $O/k12.err
echo "k12 rc=$?" >> $O/rc.txt
timeout 900 python scripts/sweep.py --max-mb 64 --out $O/sweep.md > $O/sweep.log 2>&1
echo "sweep rc=$?" >> $O/rc.txt
