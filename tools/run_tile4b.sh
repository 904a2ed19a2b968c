#!/bin/bash
# 4-GPU box: slot-major transfer order in the fused dispatch -> GEMM1; parity, then A/B
cd "$(dirname "$0")/.."
O=gpurun_out/tile4b
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_layer.py -q -x -k "tile_overlap" > $O/pytest_tile.log 2>&1
echo "tile rc=$?"; tail -1 $O/pytest_tile.log
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "layer_ep_parity and (mixtral or dsmoe or v3)" > $O/pytest_multi.log 2>&1
echo "multi rc=$?"; tail -1 $O/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() {  # name nproc tile args...
  local nm=$1 np=$2 t=$3; shift 3
  MOE_TILE_OVERLAP=$t timeout 600 $TR --nproc-per-node $np --master-port 2971$t bench.py --gpus $np "$@" > $O/${nm}_t$t.json 2> $O/${nm}_t$t.err
  python3 -c "import json;d=json.loads([l for l in open('$O/${nm}_t$t.json') if l.startswith('{')][-1]);print('$nm tile=$t', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'])" || tail -3 $O/${nm}_t$t.err
}
for r in 1 2; do for t in 1 0; do run mixtral_n4 4 $t --no-cpu-baseline --steps 30; done; done
for r in 1 2; do for t in 1 0; do run dsmoe_n4 4 $t --config dsmoe --no-cpu-baseline --steps 30; done; done
for r in 1 2; do for t in 1 0; do run dsv3_n4 4 $t --config dsv3 --no-cpu-baseline --steps 10; done; done
