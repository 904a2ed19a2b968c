#!/bin/bash
# Shared-GPU EP probe: N torchrun ranks on ONE GPU (gloo PG + CUDA IPC peer maps).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/shared
nvidia-smi --query-gpu=name,compute_mode --format=csv > gpurun_out/shared/smi.txt 2>&1
run() {  # name nproc script args...
  local name=$1 n=$2; shift 2
  local t0=$(date +%s.%N)
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
     --master-port=$((29500 + RANDOM % 1000)) "$@" > gpurun_out/shared/$name.log 2>&1
  local rc=$?
  local t1=$(date +%s.%N)
  echo "$name rc=$rc t=$(echo "$t1 - $t0" | bc) $(grep '^{' gpurun_out/shared/$name.log | tail -1 | cut -c1-300)" | tee -a gpurun_out/shared/summary.txt
}
run a2a2 2 tests/mp_a2a_worker.py
run a2a8 8 tests/mp_a2a_worker.py
run tiny8 8 tests/mp_layer_worker.py --config tiny
run mix4 4 tests/mp_layer_worker.py --config mixtral_small
run ds8 8 tests/mp_layer_worker.py --config dsmoe_small
run v3z8_dedup 8 tests/mp_layer_worker.py --config v3_small_zipf --dedup dispatch
run tiny8_graph 8 tests/mp_layer_worker.py --config tiny --graph
run pipe4 4 tests/mp_pipe_worker.py --pp 2
