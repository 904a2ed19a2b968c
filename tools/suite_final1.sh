#!/bin/bash
# 1-GPU validation at the end of the round: every GPU test, smoke, the default bench line and
# its per-phase breakdown, and the launch list of the same command.
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_final.log 2>&1; echo "pytest=$?" >> $O/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke=$?" >> $O/smoke_final.log
timeout 300 python bench.py --breakdown --steps 5 > $O/breakdown_final.log 2>&1
timeout 300 python bench.py > $O/bench_final.log 2>&1
B="python bench.py --profile-steps 2 --no-cpu-baseline"
$B > $O/plain_final.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv $B > /dev/null 2>&1
echo "ncu=$?"
