#!/bin/bash
# K1 split-length A/B: C4 (hd 128) 256 / 512 / 1024, C1 (hd 256) 256 / 512.
run() { tag=$1; cfg=$2; shift 2; env "$@" timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3i_$tag.json 2> gpurun_out/r3i_$tag.err; python -c "import json; d=json.load(open('gpurun_out/r3i_$tag.json')); print('$tag', round(d['value'],4), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; }
for i in 1 2; do
  run c4_256_$i C4 X=1; run c4_512_$i C4 IB2_K1_SPLIT=512; run c4_1024_$i C4 IB2_K1_SPLIT=1024
  run c1_256_$i C1 X=1; run c1_512_$i C1 IB2_K1_SPLIT=512
done
