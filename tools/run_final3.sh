#!/bin/bash
# HEAD validation on one B200: smoke, full pytest -m gpu, bench lines, launch list, reference
# arm; A/B of the gather launch bounds (ab/libmoe_lb.so) on DS-MoE
cd "$(dirname "$0")/.."
O=gpurun_out/final3
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
for i in 1 2; do
  timeout 600 python bench.py > $O/bench_$i.json 2> $O/bench_$i.err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_$i.json') if l.startswith('{')][-1]);print('bench', round(d['ms_per_step'],3), int(d['value']), round(d['roofline']['frac'],3), round(d['layer_roofline']['frac'],3), d['clocks']['sm_mhz'], int(d['e2e']['value']))"
done
for r in 1 2 3; do for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/ab/libmoe_lb.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/d_$V.json 2> $O/err_$V
  python3 -c "import json;d=json.loads([l for l in open('$O/d_$V.json') if l.startswith('{')][-1]);print('dsmoe $V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
unset MOE_LIB
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_mixtral.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
echo "ncu rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
