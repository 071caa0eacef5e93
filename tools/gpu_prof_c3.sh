#!/bin/bash
# C3 profiling: launch list of the bench's C3 windows, and ncu --set full of
# K2 and the CTA-pair GEMM on the C3-shaped harness.
TAG=${1:-r2}
mkdir -p gpurun_out
CFG=C3 STEPS=8 bash tools/gpu_prof_c4.sh ${TAG}_c3
timeout 300 python tools/prof_harness_c3.py > gpurun_out/${TAG}_c3h.json 2>&1; echo "harness rc=$?"; cat gpurun_out/${TAG}_c3h.json
run() {  # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c $4 \
    -o gpurun_out/${TAG}_c3_$1 python tools/prof_harness_c3.py > gpurun_out/${TAG}_c3_$1.log 2>&1
  echo "ncu $1 rc=$?"; tail -2 gpurun_out/${TAG}_c3_$1.log
}
run k2 chunk_attn_tc_kernel 16 3
run pair tc_gemm_pair_kernel 24 4
run k1 decode_attn_kernel 40 2
python tools/ncu_summary.py gpurun_out/${TAG}_c3_k2.ncu-rep gpurun_out/${TAG}_c3_pair.ncu-rep gpurun_out/${TAG}_c3_k1.ncu-rep \
  > gpurun_out/${TAG}_c3_ncu_summary.txt 2>&1
cat gpurun_out/${TAG}_c3_ncu_summary.txt
