#!/bin/bash
# 4-GPU validation at the end of the round: EP parity (plain layer, all configs, N=2/4), the
# PP x EP executor incl. its CUDA-graph replay, pipeline bench lines eager vs graph.
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "test_layer_ep_parity_dedup or test_pipeline or test_all_to_all_origin or test_layer_one_expert or (test_layer_ep_parity and not after and not chunked and not stepwise)" > $O/pytest_multi_final.log 2>&1; echo "pytest=$?" >> $O/pytest_multi_final.log
run() {  # name nproc port args...
  local name=$1 n=$2 port=$3; shift 3
  timeout 420 $TR --master-port $port --nproc-per-node $n bench.py --gpus $n "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run pipe_dsmoe_pp2ep2_graph 4 29651 --config dsmoe --pp 2 --layers 4 --micro 8 --steps 5 --warmup 3 --graph
run pipe_mixtral_pp2ep2_graph 4 29652 --pp 2 --layers 4 --micro 8 --steps 5 --warmup 3 --graph
run bench_mixtral_ep4_final 4 29653 --steps 20 --warmup 5
run bench_mixtral_ep2_final 2 29654 --steps 20 --warmup 5
