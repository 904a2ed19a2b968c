#!/bin/bash
# compute-sanitizer on the tiny layer: memcheck, racecheck, synccheck,
# initcheck on smoke() (EP = 1, fwd + bwd incl. the dedup layer) and memcheck on a 2-rank
# shared-GPU EP = 2 tiny layer (peer stores, flags).  Logs under gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
O=gpurun_out/sanitize
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
S='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 17 --print-limit 50 python -c "$S" > $O/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?" | tee -a $O/summary.txt
done
timeout 1200 $CS --tool memcheck --error-exitcode 17 --target-processes all --print-limit 50 \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29655 tests/mp_layer_worker.py --config tiny --iters 1 > $O/ep2_memcheck.log 2>&1
echo "ep2 memcheck rc=$? $(grep '^{' $O/ep2_memcheck.log | tail -1 | cut -c1-200)" | tee -a $O/summary.txt
