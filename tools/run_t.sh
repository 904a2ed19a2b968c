#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/t
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/bench_$r.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_$r.json') if l.startswith('{')][-1]);print('mixtral', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"
done
timeout 300 python bench.py --breakdown --steps 10 > $O/breakdown.json 2>&1; cut -c1-600 $O/breakdown.json
for r in 1 2; do
  timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/ds_$r.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/ds_$r.json') if l.startswith('{')][-1]);print('dsmoe', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
