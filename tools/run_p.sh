#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/p
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_symm.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "test_layer_ep_parity and (mixtral_small or dsmoe_small) and not dedup and not migration" > $O/pytest_multi.log 2>&1; echo "multi rc=$?"; tail -1 $O/pytest_multi.log
for i in 1 2; do
  timeout 300 python bench.py > $O/bench_$i.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_$i.json') if l.startswith('{')][-1]);print('bench', round(d['ms_per_step'],3), int(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['roofline']['traffic'])"
done
