#!/bin/bash
# One GPU: parity after the double-buffered wgrad epilogue, GEMM times on the V3-like slice.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q > $O/pytest_wgrad.log 2>&1 || { echo "tests failed"; tail -5 $O/pytest_wgrad.log; exit 1; }
timeout 300 python bench.py --config dsv3_slice --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_slice.log 2>&1
timeout 300 python bench.py > $O/bench1.log 2>&1
S="python bench.py --config dsv3_slice --profile-steps 1 --no-cpu-baseline"
$S > $O/plain_slice.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum --clock-control none -k regex:'grouped_gemm' --csv --log-file $O/slice_gemm_times.csv $S > /dev/null 2>&1
echo "ncu=$?"
