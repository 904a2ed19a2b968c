#!/bin/bash
# NEXT-4 evidence run (gpurun --gpus 4): dedup parity (EP=1, then N=2/4), bench lines and
# breakdowns of the fine-grained configs with the deduplicated all-to-alls.
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -k parity > $O/pytest_dedup1.log 2>&1 || { echo "ep1 tests failed"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k dedup > $O/pytest_multi_dedup.log 2>&1; echo "pytest=$?" >> $O/pytest_multi_dedup.log
run() {  # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 420 $TR --master-port $port --nproc-per-node $n bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run bench_dsv3_ep4_rebalanced_dedup 4 29621 --config dsv3 --rebalance --dedup --steps 10 --warmup 3
run breakdown_dsv3_ep4_rebalanced_dedup 4 29622 --config dsv3 --rebalance --dedup --breakdown --steps 5 --warmup 3
run bench_dsmoe_ep4_dedup 4 29623 --config dsmoe --dedup --steps 20 --warmup 5
run breakdown_dsmoe_ep4_dedup 4 29624 --config dsmoe --dedup --breakdown --steps 5 --warmup 3
run bench_dsmoe_ep2_dedup 2 29625 --config dsmoe --dedup --steps 20 --warmup 5
run bench_dsv3_ep4_dedup 4 29627 --config dsv3 --dedup --steps 10 --warmup 3
run bench_dsv3_ep4 4 29628 --config dsv3 --steps 10 --warmup 3
