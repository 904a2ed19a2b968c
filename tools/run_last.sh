#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/last
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_guard.py -q -x > $O/pytest.log 2>&1
echo "rc=$?"; tail -1 $O/pytest.log
