#!/bin/bash
# combine_bwd fused into dgrad-1: parity on one GPU
cd "$(dirname "$0")/.."
O=gpurun_out/tile2
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1 || { echo build failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x > $O/pytest_layer.log 2>&1
echo "layer rc=$?"; tail -3 $O/pytest_layer.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "layer_ep_parity or empty or collapse" > $O/pytest_multi.log 2>&1
echo "multi rc=$?"; tail -3 $O/pytest_multi.log
