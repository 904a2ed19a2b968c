#!/bin/bash
# 4-GPU box: fwd+bwd tile-granular overlap A/B (t1 = both, tb0 = forward only, t0 = off)
cd "$(dirname "$0")/.."
O=gpurun_out/tile4c
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() {  # name nproc mode args...
  local nm=$1 np=$2 m=$3; shift 3
  case $m in t1) T=1; B=1;; tb0) T=1; B=0;; t0) T=0; B=1;; esac
  MOE_TILE_OVERLAP=$T MOE_TILE_OVERLAP_BWD=$B timeout 600 $TR --nproc-per-node $np --master-port 29731 bench.py --gpus $np "$@" > $O/${nm}_$m.json 2> $O/${nm}_$m.err
  python3 -c "import json;d=json.loads([l for l in open('$O/${nm}_$m.json') if l.startswith('{')][-1]);print('$nm $m', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'], d.get('gpu_launches'))" || tail -3 $O/${nm}_$m.err
}
for r in 1 2 3; do for m in t1 tb0 t0; do run dsmoe_n4 4 $m --config dsmoe --no-cpu-baseline --steps 30; done; done
for r in 1 2; do for m in t1 t0; do run dsv3_n4 4 $m --config dsv3 --no-cpu-baseline --steps 10; done; done
for r in 1 2; do for m in t1 t0; do run mixtral_n4 4 $m --no-cpu-baseline --steps 30; done; done
