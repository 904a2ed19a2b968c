#!/bin/bash
# same-box A/B of two libmoe builds: $1 = alternative .so (MOE_LIB), $2 = bench args
cd "$(dirname "$0")/.."
O=gpurun_out/ab
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
ALT=$1; shift
for r in 1 2 3; do for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/$ALT; else unset MOE_LIB; fi
  timeout 300 python bench.py "$@" --steps 40 --no-cpu-baseline > $O/b_$V.json 2> $O/err_$V
  python3 -c "import json;d=json.loads([l for l in open('$O/b_$V.json') if l.startswith('{')][-1]);print('$V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
