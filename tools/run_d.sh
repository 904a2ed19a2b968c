#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/d
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for S in 1 0 1 0; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_s$S.json 2>$O/bench_s$S.err
  python -c "import json;d=json.load(open('$O/bench_s$S.json'));print('sched=$S', d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second"
B="python bench.py --profile-steps 2 --no-cpu-baseline"
for S in 1 0; do
MOE_GEMM_SCHED=$S timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 8 -c 8 --csv --log-file $O/ncu_s$S.csv $B > /dev/null 2>&1
echo "ncu s=$S rc=$?"
done
for c in dsmoe dsv3_slice; do
for S in 1 0; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_s$S.json 2>$O/bench_${c}_s$S.err
  python -c "import json;d=json.load(open('$O/bench_${c}_s$S.json'));print('$c sched=$S', d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done; done
