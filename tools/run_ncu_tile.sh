#!/bin/bash
# ncu --set full of the transfer-carrying GEMM launches at EP = 1 (general path: the transfer
# targets this rank's own heap), Mixtral shape; kernel replay restores memory between passes
cd "$(dirname "$0")/.."
O=gpurun_out/ncutile
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
B="python bench.py --profile-steps 2 --no-cpu-baseline"
MOE_EP1_GENERAL=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:int.5, .int.2>" -s 1 -c 1 -o $O/prof_disp_gemm1 $B > $O/ncu1.log 2>&1
echo "ncu disp rc=$?"
MOE_EP1_GENERAL=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:int.6, .int.2>" -s 1 -c 1 -o $O/prof_comb_dgrad1 $B > $O/ncu2.log 2>&1
echo "ncu comb rc=$?"
MOE_EP1_GENERAL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file $O/launches_general_tile.csv $B > /dev/null 2>&1
echo "ncu list rc=$?"
