#!/bin/bash
# same-box A/Bs: (1) EP=1 receive-layout path vs the general path, ncu launch lists (DRAM bytes
# per GEMM) + bench; (2) gather_sum launch bounds (ab/libmoe_lb.so) on DS-MoE (k = 6)
cd "$(dirname "$0")/.."
O=gpurun_out/ab2
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct"
for G in 0 1; do
  MOE_EP1_GENERAL=$G timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file $O/launches_g$G.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu general=$G rc=$?"
done
MOE_EP1_GENERAL=0 timeout 600 ncu --cache-control none --metrics $M --clock-control none -k regex:grouped_gemm --csv --log-file $O/launches_g0_nocc.csv python bench.py --profile-steps 2 --no-cpu-baseline > /dev/null 2>&1
echo "ncu nocc rc=$?"
for r in 1 2; do for G in 0 1; do
  MOE_EP1_GENERAL=$G timeout 300 python bench.py --steps 40 --no-cpu-baseline > $O/b_$G.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/b_$G.json') if l.startswith('{')][-1]);print('mixtral general=$G', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2 3; do for V in base alt; do
  if [ $V = alt ]; then export MOE_LIB=$PWD/ab/libmoe_lb.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --config dsmoe --steps 40 --no-cpu-baseline > $O/d_$V.json 2> $O/err_$V
  python3 -c "import json;d=json.loads([l for l in open('$O/d_$V.json') if l.startswith('{')][-1]);print('dsmoe $V', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
unset MOE_LIB
