#!/bin/bash
# One-GPU ncu evidence run: launch list of a Mixtral EP=1 step, --set full of the HBM-bound
# kernels (permute, unpermute, gathers, EP=1 transfers, route), --set full of the six expert
# GEMMs on the V3-like rank slice.  Every command first exits 0 without ncu.
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu1.log 2>&1; echo "pytest=$?" >> $O/pytest_gpu1.log
timeout 300 python bench.py --breakdown --steps 5 > $O/breakdown1.log 2>&1
timeout 300 python bench.py > $O/bench1.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/smoke.log
B="python bench.py --profile-steps 2 --no-cpu-baseline"
$B > $O/plain_mixtral.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mixtral_ep1.csv $B > /dev/null 2>&1
echo "launches=$?"
$B > $O/plain_mixtral2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'hist_scan|rank_kernel|scatter_kernel|gather_sum|route_kernel|transfer_kernel' -s 8 -c 8 -o $O/prof_hbm $B > /dev/null 2>&1
echo "hbm=$?"
S="python bench.py --config dsv3_slice --profile-steps 1 --no-cpu-baseline"
$S > $O/plain_slice.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'grouped_gemm' -s 1 -c 6 -o $O/prof_slice_gemm $S > /dev/null 2>&1
echo "slice=$?"
D="python bench.py --config dsmoe --dedup all --profile-steps 2 --no-cpu-baseline"
$D > $O/plain_dedup.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'dedup' -s 9 -c 9 -o $O/prof_dedup $D > /dev/null 2>&1
echo "dedup=$?"
