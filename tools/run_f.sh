#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/f
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
timeout 300 python bench.py --breakdown --steps 10 > $O/breakdown.json 2>&1; cut -c1-900 $O/breakdown.json
for c in mixtral dsmoe; do for P in 1 0 1 0; do
  MOE_GEMM_PAIR=$P timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_p$P.json 2>$O/bench_${c}_p$P.err
  python -c "import json;d=json.load(open('$O/bench_${c}_p$P.json'));print('$c pair=$P', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done; done
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
B="python bench.py --profile-steps 2 --no-cpu-baseline"
for X in 0 1; do
  if [ $X = 1 ]; then export MOE_DBG_NO_AUX=1; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 11 -c 1 --csv --log-file $O/ncu_dgrad1_noaux$X.csv $B > /dev/null 2>&1
  echo "ncu noaux=$X rc=$?"
done
unset MOE_DBG_NO_AUX
