#!/bin/bash
# 4-GPU box, final HEAD: multi-rank suite over NCCL (EP = 8 shares 2 ranks per GPU) and bench
# lines at the final defaults
cd "$(dirname "$0")/.."
O=gpurun_out/final4
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
line() { python3 -c "import json;d=json.loads([l for l in open('$1') if l.startswith('{')][-1]);print('$2', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'], d.get('gpu_launches'))" || tail -3 $1.err; }
for n in 2 4; do
  timeout 600 $TR --nproc-per-node $n --master-port 2975$n bench.py --gpus $n --no-cpu-baseline > $O/mixtral_n$n.json 2> $O/mixtral_n$n.json.err; line $O/mixtral_n$n.json mixtral_n$n
  timeout 600 $TR --nproc-per-node $n --master-port 2976$n bench.py --gpus $n --config dsmoe --no-cpu-baseline > $O/dsmoe_n$n.json 2> $O/dsmoe_n$n.json.err; line $O/dsmoe_n$n.json dsmoe_n$n
done
timeout 900 $TR --nproc-per-node 4 --master-port 29771 bench.py --gpus 4 --config dsv3 --steps 10 --no-cpu-baseline > $O/dsv3_n4.json 2> $O/dsv3_n4.json.err; line $O/dsv3_n4.json dsv3_n4
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -x -rs > $O/pytest_multi.log 2>&1
echo "multi rc=$?"; tail -3 $O/pytest_multi.log
