#!/bin/bash
# Multi-GPU evidence run (gpurun --gpus 4): EP parity tests, bench lines and per-phase
# breakdowns at N=2/4.  Outputs land in gpurun_out/ (copy the keepers to profiles/rNN/).
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_multi.log 2>&1; echo "pytest=$?" >> $O/pytest_multi.log
run() {  # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 420 $TR --master-port $port --nproc-per-node $n bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run bench_mixtral_ep2 2 29611 --steps 20 --warmup 5
run bench_mixtral_ep4 4 29612 --steps 20 --warmup 5
run bench_dsmoe_ep4 4 29613 --config dsmoe --steps 20 --warmup 5
run bench_dsv3_ep4_rebalanced 4 29614 --config dsv3 --rebalance --steps 10 --warmup 3
run breakdown_dsv3_ep4_rebalanced 4 29615 --config dsv3 --rebalance --breakdown --steps 5 --warmup 3
run breakdown_dsmoe_ep4 4 29616 --config dsmoe --breakdown --steps 5 --warmup 3
run breakdown_mixtral_ep4 4 29617 --breakdown --steps 5 --warmup 3
