#!/bin/bash
# 4-GPU box: multi-rank parity on real GPUs (EP=8 as 2 ranks per GPU), bench lines at N=2/4,
# the config-5 all-to-all sweeps at N=2/4.  Logs under gpurun_out/multi/.
cd "$(dirname "$0")/.."
O=gpurun_out/multi
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for N in 2 4; do
  timeout 600 $TR --nproc-per-node $N --master-port 29610 bench.py --gpus $N > $O/bench_mixtral_n$N.json 2> $O/bench_mixtral_n$N.err
  echo "mixtral N=$N rc=$? $(cut -c1-200 $O/bench_mixtral_n$N.json)"
done
timeout 600 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config dsmoe --dedup > $O/bench_dsmoe_n4_dedup.json 2> $O/bench_dsmoe_n4.err
echo "dsmoe rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --config dsv3 --rebalance --steps 20 > $O/bench_dsv3_n4_rebal.json 2> $O/bench_dsv3_n4.err
echo "dsv3 rc=$?"
for N in 2 4; do
  timeout 900 $TR --nproc-per-node $N --master-port 29613 bench.py --gpus $N --a2a > $O/a2a_sweep_n$N.json 2> $O/a2a_n$N.err
  echo "a2a N=$N rc=$?"
done
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -x -rs > $O/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; tail -3 $O/pytest_multi.log
