#!/bin/bash
# NEXT-1 tile-granular dispatch -> GEMM1: parity on one GPU (EP = 1 general path, then EP = 2/4/8
# ranks sharing the GPU), then same-box timing of the A/Bs
cd "$(dirname "$0")/.."
O=gpurun_out/tile
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1 || { echo build failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -k "tile_overlap" > $O/pytest_tile.log 2>&1
echo "tile rc=$?"; tail -3 $O/pytest_tile.log
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multi.py -q -x -k "fused or local_path or layer_ep_parity or empty" > $O/pytest_multi.log 2>&1
echo "multi rc=$?"; tail -3 $O/pytest_multi.log
bash tools/run_ab2.sh
