#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/b
python paper_2605_05049_b200/build.py > gpurun_out/b/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "empty or local_path or origin_encoded or pipeline or collapse or placement or fused_and_stepwise" > gpurun_out/b/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b/pytest.log
tail -2 gpurun_out/b/pytest.log
timeout 600 python bench.py > gpurun_out/b/bench.json 2> gpurun_out/b/bench.err
echo "bench rc=$?"; cut -c1-400 gpurun_out/b/bench.json
HINTS="0 1 3 7" bash tools/exp_l2.sh
