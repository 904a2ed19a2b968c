#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/g
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$i.json 2>$O/bench_$i.err
  python -c "import json;d=json.load(open('$O/bench_$i.json'));print('mixtral', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['e2e']['value'])"
done
for i in 1 2; do
  timeout 300 python bench.py --config dsmoe --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_ds_$i.json 2>$O/bench_ds_$i.err
  python -c "import json;d=json.load(open('$O/bench_ds_$i.json'));print('dsmoe', round(d['ms_per_step'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])"
done
B="python bench.py --profile-steps 2 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>&1
echo "ncu rc=$?"
