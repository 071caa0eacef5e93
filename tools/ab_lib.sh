#!/bin/bash
# A/B of two builds of the library on one box: _ab/new and _ab/old hold the .so variants.
# Usage (GPU box): bash tools/ab_lib.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fused_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fused_pytest.log
for v in new old new old; do
  cp _ab/$v/libinfercept_b200.so paper_2402_01869_b200/
  timeout 400 python bench.py --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/ab_$v.json').read().splitlines()[-1])
print('$v', 'req/s %.3f ms/step %.3f K1 %.0f GB/s frac %.3f' % (j['value'], j['ms_per_step'], j['roofline']['achieved'], j['roofline']['frac']), j['clocks']['sm_mhz'])"
done
