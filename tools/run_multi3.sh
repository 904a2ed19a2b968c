#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/multi3
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k dsmoe > $O/pytest_full.log 2>&1
echo "pytest full rc=$?"; tail -1 $O/pytest_full.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
for S in 1 0 1 0; do
  MOE_GEMM_SCHED=$S timeout 600 $TR --nproc-per-node 4 --master-port 29610 bench.py --gpus 4 > $O/bench_mixtral_n4_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_mixtral_n4_s$S.json') if l.startswith('{')][-1]);print('mixtral n4 sched=$S', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), d['clocks']['sm_mhz'])"
done
for S in 1 0; do
  MOE_GEMM_SCHED=$S timeout 600 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config dsmoe > $O/bench_dsmoe_n4_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_dsmoe_n4_s$S.json') if l.startswith('{')][-1]);print('dsmoe n4 sched=$S', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), d['clocks']['sm_mhz'])"
done
for S in 1 0; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --config dsmoe --steps 30 --no-cpu-baseline > $O/bench_dsmoe_n1_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_dsmoe_n1_s$S.json') if l.startswith('{')][-1]);print('dsmoe n1 sched=$S', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), d['clocks']['sm_mhz'])"
done
