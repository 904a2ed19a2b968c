#!/bin/bash
# 4-GPU box: V3-like N=4 after migration: tile-granular transfers vs the dedup all-to-all
cd "$(dirname "$0")/.."
O=gpurun_out/v3mig
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node 4 --master-port 29741"
run() {
  local nm=$1; shift
  timeout 900 $TR bench.py --gpus 4 --config dsv3 --no-cpu-baseline --steps 10 "$@" > $O/$nm.json 2> $O/$nm.err
  python3 -c "import json;d=json.loads([l for l in open('$O/$nm.json') if l.startswith('{')][-1]);print('$nm', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'])" || tail -3 $O/$nm.err
}
for r in 1 2; do
  run mig_tile --rebalance
  MOE_TILE_OVERLAP=0 run mig_sep --rebalance
  run mig_dedup --rebalance --dedup
done
