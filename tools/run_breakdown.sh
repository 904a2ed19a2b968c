#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/bd
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 300 python bench.py --breakdown --steps 20 --no-cpu-baseline > $O/breakdown_mixtral.json 2> $O/err1; echo "rc=$?"
timeout 300 python bench.py --config dsmoe --breakdown --steps 20 --no-cpu-baseline > $O/breakdown_dsmoe.json 2> $O/err2; echo "rc=$?"
tail -c 1500 $O/breakdown_mixtral.json
