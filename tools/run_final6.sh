#!/bin/bash
# last full validation of the round's HEAD on one B200
cd "$(dirname "$0")/.."
O=gpurun_out/final6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 20 > $O/bench.json 2> $O/bench.err
python3 -c "import json;d=json.loads([l for l in open('$O/bench.json') if l.startswith('{')][-1]);print('bench', round(d['ms_per_step'],3), int(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
timeout 3000 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
