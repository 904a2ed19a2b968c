#!/bin/bash
# dSwiGLU epilogue with 2 staging boxes (default build) vs 1 (ab/libmoe_dsw1.so): parity of the
# default build, then alternating benches + dgrad-1 launch metrics
cd "$(dirname "$0")/.."
O=gpurun_out/dsw
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2 3; do for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/ab/libmoe_dsw1.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/b_$V.json 2> $O/err_$V
  python3 -c "import json;d=json.loads([l for l in open('$O/b_$V.json') if l.startswith('{')][-1]);print('mixtral $V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2; do for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/ab/libmoe_dsw1.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/d_$V.json 2> $O/errd_$V
  python3 -c "import json;d=json.loads([l for l in open('$O/d_$V.json') if l.startswith('{')][-1]);print('dsmoe $V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/ab/libmoe_dsw1.so; else unset MOE_LIB; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file $O/launches_$V.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $V rc=$?"
done
