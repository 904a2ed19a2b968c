#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/n
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr=127.0.0.1 --master-port=29777 tests/mp_layer_worker.py --config dsmoe_small > $O/ds8.log 2>&1
echo "ds8 rc=$?"; grep -n "Error\|error" $O/ds8.log | head -20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29778 tests/mp_layer_worker.py --config dsmoe_small > $O/ds2.log 2>&1
echo "ds2 rc=$?"; grep -n "Error\|error\|^{" $O/ds2.log | head -10 | cut -c1-300
