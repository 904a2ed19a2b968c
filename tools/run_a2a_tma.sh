#!/bin/bash
# config-5 sweep: static all-to-all with SM stores vs TMA bulk copies, N=2 and N=4
cd "$(dirname "$0")/.."
O=gpurun_out/a2a_tma
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for N in 4 2; do for T in 1 0; do
  MOE_A2A_TMA=$T timeout 900 $TR --nproc-per-node $N --master-port 2962$T bench.py --gpus $N --a2a > $O/a2a_n${N}_tma$T.json 2> $O/a2a_n${N}_tma$T.err
  echo "a2a N=$N tma=$T rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "origin_encoded" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
MOE_A2A_TMA=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "origin_encoded" > $O/pytest_tma.log 2>&1; tail -1 $O/pytest_tma.log
