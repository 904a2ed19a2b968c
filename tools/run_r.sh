#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "migration or pipeline" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
