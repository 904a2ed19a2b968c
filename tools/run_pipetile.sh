#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/pipetile
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_layer.py -q -x -k "pipeline or tile_overlap" > $O/pytest.log 2>&1
echo "rc=$?"; tail -2 $O/pytest.log
