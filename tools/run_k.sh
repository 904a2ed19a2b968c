#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/k
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
for r in 1 2; do for S in 0 1 2 3; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --config dsmoe --steps 30 --no-cpu-baseline > $O/bench_dsmoe_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_dsmoe_s$S.json') if l.startswith('{')][-1]);print('dsmoe sched=$S', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
for r in 1 2; do for S in 0 1 3; do
  MOE_GEMM_SCHED=$S timeout 300 python bench.py --steps 30 --no-cpu-baseline > $O/bench_mixtral_s$S.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/bench_mixtral_s$S.json') if l.startswith('{')][-1]);print('mixtral sched=$S', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
