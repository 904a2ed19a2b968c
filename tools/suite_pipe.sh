#!/bin/bash
# NEXT-3 evidence run (gpurun --gpus 4): PP x EP executor parity, then bench lines.
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -k pipeline > $O/pytest_pipe.log 2>&1; echo "pytest=$?" >> $O/pytest_pipe.log
grep -q "pytest=0" $O/pytest_pipe.log || exit 1
run() {  # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 420 $TR --master-port $port --nproc-per-node $n bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run pipe_dsmoe_pp2ep2 4 29641 --config dsmoe --pp 2 --layers 4 --micro 8 --steps 5 --warmup 3
run pipe_dsmoe_pp4ep1 4 29642 --config dsmoe --pp 4 --layers 4 --micro 8 --steps 5 --warmup 3
run pipe_mixtral_pp2ep2 4 29643 --pp 2 --layers 4 --micro 8 --steps 5 --warmup 3
