#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r2d; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "zero_filling or selected_unpack or overlapped or multi_rank_code or ddp_hook or peer or host_pipeline or fp32_full" > $O/pytest_sel.log 2>&1
echo "pytest rc=$?" > $O/rc.txt
NAMES="base k2w2" timeout 900 bash scripts/variants.sh k12 > $O/k12_variants.jsonl 2> $O/k12.err
echo "k12 rc=$?" >> $O/rc.txt
timeout 900 python scripts/sweep.py --max-mb 64 --out $O/sweep.md > $O/sweep.log 2>&1
echo "sweep rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/rc.txt
timeout 1500 python scripts/real_models.py --models resnet50,vgg16,bert_large --intervals 1,4 > $O/real_models.jsonl 2> $O/real_models.err
echo "real rc=$?" >> $O/rc.txt
