#!/bin/bash
# L2 eviction-policy experiment on the Mixtral EP=1 step: bench line + per-launch DRAM bytes,
# time and tensor-pipe activity of every grouped-GEMM launch of one step, per MOE_L2_HINT.
cd "$(dirname "$0")/.."
O=gpurun_out/l2
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct"
for H in ${HINTS:-0 1 3 7 2 6}; do
  MOE_L2_HINT=$H timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_h$H.json 2> $O/bench_h$H.err
  B="python bench.py --profile-steps 2 --no-cpu-baseline"
  MOE_L2_HINT=$H timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 8 -c 8 --csv \
     --log-file $O/ncu_h$H.csv $B > /dev/null 2>&1
  echo "h=$H rc=$? $(python -c "import json;d=json.load(open('$O/bench_h$H.json'));print(d['ms_per_step'],d['clocks'])" 2>&1)"
done
