#!/bin/bash
# same-box A/B: libmoe.so (GEMM setup before griddepcontrol.wait) vs libmoe_ab.so (HEAD~)
cd "$(dirname "$0")/.."
O=gpurun_out/q
mkdir -p $O
for r in 1 2 3; do for V in new old; do
  if [ $V = old ]; then export MOE_LIB=$PWD/paper_2605_05049_b200/libmoe_ab.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/bench_$V.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_$V.json') if l.startswith('{')][-1]);print('$V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
unset MOE_LIB
for r in 1 2; do for V in new old; do
  if [ $V = old ]; then export MOE_LIB=$PWD/paper_2605_05049_b200/libmoe_ab.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/ds_$V.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/ds_$V.json') if l.startswith('{')][-1]);print('ds $V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
