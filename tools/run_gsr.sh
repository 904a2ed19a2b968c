#!/bin/bash
# permute_bwd + router gather: all loads of an iteration before the first use (default build)
# vs the committed two-phase kernel (ab/libmoe_base.so); parity of the default build first
cd "$(dirname "$0")/.."
O=gpurun_out/gsr
mkdir -p $O
python paper_2605_05049_b200/build.py > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2; do for V in new base; do
  if [ $V = base ]; then export MOE_LIB=$PWD/ab/libmoe_base.so; else unset MOE_LIB; fi
  timeout 300 python bench.py --config dsmoe --breakdown --steps 20 --no-cpu-baseline > $O/d_$V.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/d_$V.json') if l.startswith('{')][-1]);b=d['breakdown_ms_max_over_ranks'];print('dsmoe $V', b['B2 permute_bwd'], b['F6 unpermute'], round(d['sum_ms'],3))"
  timeout 300 python bench.py --breakdown --steps 20 --no-cpu-baseline > $O/m_$V.json 2> $O/err
  python3 -c "import json;d=json.loads([l for l in open('$O/m_$V.json') if l.startswith('{')][-1]);b=d['breakdown_ms_max_over_ranks'];print('mixtral $V', b['B2 permute_bwd'], b['F6 unpermute'], round(d['sum_ms'],3))"
done; done
unset MOE_LIB
