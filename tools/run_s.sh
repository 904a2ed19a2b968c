#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
B="python bench.py --profile-steps 2 --no-cpu-baseline"
for X in 1 0; do
  MOE_DSWIGLU_TMA=$X timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm -s 11 -c 1 --csv --log-file $O/dgrad1_t$X.csv $B > /dev/null 2>&1
  echo "ncu t=$X rc=$?"
done
for r in 1 2 3; do for X in 1 0; do
  MOE_DSWIGLU_TMA=$X timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/bench_t$X.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_t$X.json') if l.startswith('{')][-1]);print('mixtral tma=$X', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2; do for X in 1 0; do
  MOE_DSWIGLU_TMA=$X timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/ds_t$X.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/ds_t$X.json') if l.startswith('{')][-1]);print('dsmoe tma=$X', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
