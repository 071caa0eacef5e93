#!/bin/bash
# A/B of an executor env switch on the bench (same box, alternating runs).
# Usage: gpurun -- 'AB_ENV=IB2_NO_SPLIT_BATCH=1 bash tools/gpu_ab.sh TAG [bench args]'
TAG=$1; shift
ARGS=${@:---steps 20 --warmup 5 --no-cpu-baseline}
mkdir -p gpurun_out
for i in 1 2; do
  timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_A$i.json 2>gpurun_out/${TAG}_A$i.err
  env $AB_ENV timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_B$i.json 2>gpurun_out/${TAG}_B$i.err
done
for f in gpurun_out/${TAG}_A1 gpurun_out/${TAG}_B1 gpurun_out/${TAG}_A2 gpurun_out/${TAG}_B2; do
  python -c "import json,sys; d=json.load(open('$f.json')); print('$f', round(d['value'],4), 'ms/step', round(d['ms_per_step'],2), 'k1', round(d['roofline']['frac'],3), 'step_roof', round(d['step_roofline']['frac'],3))" 2>&1 | tail -1
  tail -2 $f.err
done
