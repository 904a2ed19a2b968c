#!/bin/bash
# static vs dynamic GEMM tile schedule (8-slot queue), alternating, N=4 and N=1, one box
cd "$(dirname "$0")/.."
O=gpurun_out/multi5
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for r in 1 2 3; do for S in 0 1; do
  MOE_GEMM_SCHED=$S timeout 600 $TR --nproc-per-node 4 --master-port 2962$S bench.py --gpus 4 > $O/n4_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/n4_s$S.json') if l.startswith('{')][-1]);print('n4 sched=$S', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2 3; do for S in 0 1; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/n1_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/n1_s$S.json') if l.startswith('{')][-1]);print('n1 sched=$S', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
