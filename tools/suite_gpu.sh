#!/bin/bash
# Full GPU suite on one box: pytest -m gpu (multi-rank cases share the GPU when it has fewer
# GPUs than ranks, tests/mp_common.py) + smoke(); logs under gpurun_out/suite/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/suite
python paper_2605_05049_b200/build.py > gpurun_out/suite/build.log 2>&1
start=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q -x -rs --durations=30 ${PYTEST_ARGS} > gpurun_out/suite/pytest.log 2>&1
echo "pytest rc=$? elapsed=$(( $(date +%s) - start ))s" >> gpurun_out/suite/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/suite/smoke.log 2>&1
tail -3 gpurun_out/suite/pytest.log
