#!/bin/bash
# The multi-GPU evidence this repository still owes, in one call, for the
# first box with P >= 2 GPUs (one process per GPU):
#   * the multi-GPU test cases (NCCL sync, NCCL-window peer with and without
#     the NVSwitch multimem reduction) — skipped below P devices;
#   * bench.py at N = 2, 4, 8 (the driver's SCALE contract) with the default
#     NCCL collective, the rank-ordered peer collective, the NCCL-window peer
#     with multimem, the symmetric send window and pipelined bucket groups;
#   * the allreduce / sync-step sweep (roofline.c1 vs 900 GB/s).
# Output under gpurun_out/${1:-multi}.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-multi}; mkdir -p $O
G=$(python -c "import torch; print(torch.cuda.device_count())")
echo "gpus=$G" | tee $O/rc.txt
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 2400 python -m pytest tests/test_multiproc.py -q -m gpu -rs > $O/pytest_multiproc.log 2>&1
echo "multiproc tests rc=$?" | tee -a $O/rc.txt
run() {  # N, label, extra bench args
  local N=$1 L=$2; shift 2
  [ "$N" -le "$G" ] || return 0
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline "$@" \
    >> $O/bench_$L.jsonl 2>> $O/bench_$L.err
  echo "bench $L N=$N rc=$?" | tee -a $O/rc.txt
}
for N in 2 4 8; do
  run $N nccl
  run $N nccl_auto --interval auto
  run $N peer --collective peer --no-real-model --no-overhead
  run $N peer_window --collective peer --peer-window --no-real-model --no-overhead
  run $N multimem --collective peer --peer-window --multimem --no-real-model --no-overhead
  run $N symmetric --symmetric --no-real-model --no-overhead
  run $N pipeline4 --pipeline 4 --no-real-model --no-overhead
  run $N pipeline4_free16 --pipeline 4 --free-sms 16 --no-real-model --no-overhead
  run $N overlap_free16 --free-sms 16 --no-real-model
  run $N bert --layout bert_large --interval 4 --no-real-model
done
if [ "$G" -ge 2 ]; then
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 \
    --master-port 29600 scripts/nccl_sweep.py --out $O/nccl_sweep.jsonl > $O/nccl_sweep.log 2>&1
  echo "nccl sweep rc=$?" | tee -a $O/rc.txt
fi
