#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/c
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "empty or local_path or origin_encoded or pipeline or collapse or placement or fused_and_stepwise" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
B="python bench.py --profile-steps 2 --no-cpu-baseline"
$B > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 11 -c 1 -o $O/prof_dgrad1 $B > $O/ncu1.log 2>&1
echo "ncu dgrad1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 13 -c 1 -o $O/prof_wgrad $B > $O/ncu2.log 2>&1
echo "ncu wgrad rc=$?"
bash tools/sanitize.sh
