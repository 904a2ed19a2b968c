#!/bin/bash
# 4-GPU run: EP=1 parity after the gather-kernel rewrite, then the SM budget of the
# all-to-all running beside the shared-expert GEMMs (DS-MoE N=4), plain vs dedup.
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -x -q > $O/pytest_ep1.log 2>&1 || { echo "ep1 tests failed"; exit 1; }
run() {  # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 420 $TR --master-port $port --nproc-per-node $n bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run sms_dsmoe_plain_20 4 29631 --config dsmoe --steps 20 --warmup 5 --comm-sms 20
run sms_dsmoe_plain_48 4 29632 --config dsmoe --steps 20 --warmup 5 --comm-sms 48
run sms_dsmoe_dedup_20 4 29633 --config dsmoe --dedup --steps 20 --warmup 5 --comm-sms 20
run sms_dsmoe_dedup_48 4 29634 --config dsmoe --dedup --steps 20 --warmup 5 --comm-sms 48
run sms_dsmoe_dedup_74 4 29635 --config dsmoe --dedup --steps 20 --warmup 5 --comm-sms 74
run sms_mixtral_ep4 4 29636 --steps 20 --warmup 5
run sms_mixtral_ep2 2 29637 --steps 20 --warmup 5
