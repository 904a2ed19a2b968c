#!/bin/bash
# same-box A/B: EP=1 in place (default) vs the general permute + dispatch + fused-scatter path
cd "$(dirname "$0")/.."
O=gpurun_out/u
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
for r in 1 2 3; do for G in 0 1; do
  MOE_EP1_GENERAL=$G timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/b_$G.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/b_$G.json') if l.startswith('{')][-1]);print('mixtral general=$G', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2; do for G in 0 1; do
  MOE_EP1_GENERAL=$G timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/d_$G.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/d_$G.json') if l.startswith('{')][-1]);print('dsmoe general=$G', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
