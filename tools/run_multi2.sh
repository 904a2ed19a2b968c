#!/bin/bash
# 4-GPU box, current HEAD: bench lines at N=2/4 (Mixtral), DS-MoE / V3-like at N=4, breakdowns
cd "$(dirname "$0")/.."
O=gpurun_out/multi2
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for N in 2 4; do
  timeout 600 $TR --nproc-per-node $N --master-port 29610 bench.py --gpus $N > $O/bench_mixtral_n$N.json 2> $O/bench_mixtral_n$N.err
  echo "mixtral N=$N rc=$?"
done
timeout 600 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config dsmoe > $O/bench_dsmoe_n4.json 2> $O/bench_dsmoe_n4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --config dsmoe --dedup > $O/bench_dsmoe_n4_dedup.json 2> $O/bench_dsmoe_n4_dedup.err
timeout 900 $TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --config dsv3 --rebalance --steps 20 > $O/bench_dsv3_n4_rebal.json 2> $O/bench_dsv3_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --config dsv3 --rebalance --dedup --steps 20 > $O/bench_dsv3_n4_rebal_dedup.json 2> $O/bench_dsv3_n4_dedup.err
timeout 600 $TR --nproc-per-node 4 --master-port 29615 bench.py --gpus 4 --breakdown --steps 10 > $O/breakdown_mixtral_n4.json 2> $O/breakdown_mixtral_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29616 bench.py --gpus 4 --pp 2 --graph > $O/pipe_mixtral_pp2ep2.json 2> $O/pipe.err
for f in $O/*.json; do echo "$f $(grep '^{' $f | tail -1 | cut -c1-150)"; done
