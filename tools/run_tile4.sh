#!/bin/bash
# 4-GPU box: NEXT-1 tile-granular dispatch -> GEMM1 (MOE_TILE_OVERLAP=1, default) against the
# separate dispatch + GEMM1 (=0), alternating on one box; then the multi-rank parity tests
# over NCCL (one GPU per rank; EP = 8 shares 2 ranks per GPU)
cd "$(dirname "$0")/.."
O=gpurun_out/tile4
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() {  # name nproc tile args...
  local nm=$1 np=$2 t=$3; shift 3
  MOE_TILE_OVERLAP=$t timeout 600 $TR --nproc-per-node $np --master-port 2971$t bench.py --gpus $np "$@" > $O/${nm}_t$t.json 2> $O/${nm}_t$t.err
  python3 -c "import json;d=json.loads([l for l in open('$O/${nm}_t$t.json') if l.startswith('{')][-1]);print('$nm tile=$t', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'], d.get('gpu_launches'))" || tail -3 $O/${nm}_t$t.err
}
for r in 1 2; do for t in 1 0; do run mixtral_n4 4 $t --no-cpu-baseline; done; done
for r in 1 2; do for t in 1 0; do run mixtral_n2 2 $t --no-cpu-baseline; done; done
for r in 1 2; do for t in 1 0; do run dsmoe_n4 4 $t --config dsmoe --no-cpu-baseline; done; done
for r in 1 2; do for t in 1 0; do run dsv3_n4 4 $t --config dsv3 --no-cpu-baseline --steps 20; done; done
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "layer_ep_parity or pipeline" > $O/pytest_multi.log 2>&1
echo "multi rc=$?"; tail -3 $O/pytest_multi.log
