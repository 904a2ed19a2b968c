#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/j
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
MOE_EPI_HALVES=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > $O/pytest_eh1.log 2>&1
echo "pytest eh1 rc=$?" >> $O/pytest_eh1.log; tail -1 $O/pytest_eh1.log
for c in mixtral dsmoe; do for H in 2 1 2 1; do
  MOE_EPI_HALVES=$H timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_h$H.json 2>$O/bench_${c}_h$H.err
  python -c "import json;d=json.load(open('$O/bench_${c}_h$H.json'));print('$c halves=$H', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for H in 2 1; do
B="python bench.py --profile-steps 2 --no-cpu-baseline"
MOE_EPI_HALVES=$H timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 8 -c 8 --csv --log-file $O/ncu_h$H.csv $B > /dev/null 2>&1
echo "ncu h=$H rc=$?"
done
