#!/bin/bash
# 1-GPU validation at the end of the round: every GPU test, smoke, the default bench line.
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_final.log 2>&1; echo "pytest=$?" >> $O/pytest_gpu_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke=$?" >> $O/smoke_final.log
timeout 240 python bench.py > $O/bench_final.log 2>&1; echo "bench=$?" >> $O/bench_final.log
tail -2 $O/pytest_gpu_final.log; tail -2 $O/smoke_final.log; tail -1 $O/bench_final.log
