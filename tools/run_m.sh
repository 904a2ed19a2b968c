#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/m
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "test_layer_ep_parity and (dsmoe_small or v3_small_zipf) and not dedup and not migration" > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -1 $O/pytest_multi.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in dsmoe mixtral; do
  B="python bench.py --config $c --profile-steps 2 --no-cpu-baseline"
  timeout 600 ncu --metrics $M --clock-control none -k regex:'transfer|gather|scatter' --csv --log-file $O/hbm_$c.csv $B > /dev/null 2>&1
  echo "ncu $c rc=$?"
done
for c in dsmoe mixtral; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > $O/bench_$c.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_$c.json') if l.startswith('{')][-1]);print('$c', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
B="python bench.py --profile-steps 2 --no-cpu-baseline"
for X in 0 1; do
  if [ $X = 1 ]; then export MOE_DGRAD2_NFAST=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:grouped_gemm -s 12 -c 1 --csv --log-file $O/dgrad2_nf$X.csv $B > /dev/null 2>&1
  echo "ncu dgrad2 nf=$X rc=$?"
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --no-cpu-baseline > $O/bench_nf$X.json 2> $O/err
    python3 -c "import json;d=json.loads([l for l in open('$O/bench_nf$X.json') if l.startswith('{')][-1]);print('mixtral nf=$X', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  done
done
unset MOE_DGRAD2_NFAST
