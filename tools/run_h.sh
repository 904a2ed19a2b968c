#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/h
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "test_layer_ep_parity and (mixtral_small or dsmoe_small or drops) and not dedup and not migration" > $O/pytest_multi.log 2>&1
echo "pytest multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
for c in mixtral dsmoe; do for T in 1 0 1 0; do
  MOE_GEMM_TAILS=$T timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_${c}_t$T.json 2>$O/bench_${c}_t$T.err
  python -c "import json;d=json.load(open('$O/bench_${c}_t$T.json'));print('$c tails=$T', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done; done
B="python bench.py --profile-steps 2 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>&1
echo "ncu rc=$?"
