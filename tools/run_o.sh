#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/o
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
B="python bench.py --profile-steps 2 --no-cpu-baseline"
for X in 0 1; do
  if [ $X = 1 ]; then export MOE_DGRAD2_NFAST=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:grouped_gemm -s 12 -c 1 --csv --log-file $O/dgrad2_nf$X.csv $B > /dev/null 2>&1
  echo "ncu dgrad2 nf=$X rc=$?"
done
unset MOE_DGRAD2_NFAST
for r in 1 2; do for X in 0 1; do
  if [ $X = 1 ]; then export MOE_DGRAD2_NFAST=1; else unset MOE_DGRAD2_NFAST; fi
  timeout 300 python bench.py --steps 30 --no-cpu-baseline > $O/bench_nf$X.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_nf$X.json') if l.startswith('{')][-1]);print('mixtral nf=$X', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
