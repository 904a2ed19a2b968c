#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/i
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for c in dsmoe dsv3_slice; do
  B="python bench.py --config $c --profile-steps 2 --no-cpu-baseline"
  $B > $O/plain_$c.log 2>&1
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$c.csv $B > /dev/null 2>&1
  echo "ncu $c rc=$?"
done
timeout 300 python bench.py --config dsmoe --breakdown --steps 10 > $O/breakdown_dsmoe.json 2>&1; cut -c1-700 $O/breakdown_dsmoe.json
