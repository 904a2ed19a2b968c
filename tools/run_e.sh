#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/e
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for S in 1 0 1 0 1 0; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_s$S.json 2>$O/bench_s$S.err
  python -c "import json;d=json.load(open('$O/bench_s$S.json'));print('sched=$S', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks'])"
done
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,sm__cycles_elapsed.avg"
B="python bench.py --profile-steps 2 --no-cpu-baseline"
MOE_GEMM_SCHED=1 timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 8 -c 8 --csv --log-file $O/ncu_s1.csv $B > /dev/null 2>&1
echo "ncu rc=$?"
