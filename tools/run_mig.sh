#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/mig
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for N in 2 4; do for c in mixtral dsv3; do
  timeout 900 $TR --nproc-per-node $N --master-port 2963$N bench.py --gpus $N --migrate-bench --config $c --steps 5 --warmup 2 > $O/mig_${c}_n$N.json 2> $O/mig_${c}_n$N.err
  echo "$c N=$N rc=$? $(grep '^{' $O/mig_${c}_n$N.json | cut -c1-400)"
done; done
