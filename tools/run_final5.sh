#!/bin/bash
# Final HEAD on a 2-GPU box: smoke, bench N=1 and N=2 (Mixtral, DS-MoE), full pytest -m gpu
cd "$(dirname "$0")/.."
O=gpurun_out/final5
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
line() { python3 -c "import json;d=json.loads([l for l in open('$1') if l.startswith('{')][-1]);print('$2', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'], d.get('gpu_launches'), d['config'].get('tile_overlap'), round(d['roofline']['frac'],3))" || tail -3 $1.err; }
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.json.err; line $O/bench_n1.json mixtral_n1
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 29781 bench.py --gpus 2 > $O/mixtral_n2.json 2> $O/mixtral_n2.json.err; line $O/mixtral_n2.json mixtral_n2
timeout 600 $TR --master-port 29782 bench.py --gpus 2 --config dsmoe --no-cpu-baseline > $O/dsmoe_n2.json 2> $O/dsmoe_n2.json.err; line $O/dsmoe_n2.json dsmoe_n2
timeout 600 $TR --master-port 29783 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > $O/ref_n2.json 2> $O/ref_n2.json.err; tail -c 300 $O/ref_n2.json
timeout 3000 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
