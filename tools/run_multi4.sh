#!/bin/bash
# 4-GPU box, HEAD: the multi-rank suite on real GPUs (EP=8 as 2 ranks per GPU; the PP x EP
# CUDA-graph case with NCCL hand-offs), bench lines at N=2/4.
cd "$(dirname "$0")/.."
O=gpurun_out/multi4
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for N in 2 4; do for r in 1 2; do
  timeout 600 $TR --nproc-per-node $N --master-port 2961$r bench.py --gpus $N > $O/bench_mixtral_n${N}_$r.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_mixtral_n${N}_$r.json') if l.startswith('{')][-1]);print('mixtral n$N', round(d['ms_per_step'],3), int(d['value']), round(d['layer_roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
timeout 2700 python -m pytest tests/test_gpu_multi.py -q -x -rs > $O/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; tail -3 $O/pytest_multi.log
