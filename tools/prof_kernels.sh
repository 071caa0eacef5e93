#!/bin/bash
# ncu --set full captures of the hot kernels on the small-pool harness
# (tools/prof_harness.py): fast replays, shapes of the C1 window.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 120 python tools/prof_harness.py > gpurun_out/${TAG}_harness.json 2>&1; echo "harness rc=$?"; cat gpurun_out/${TAG}_harness.json
run() {  # name regex skip count
  timeout 420 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c $4 \
    -o gpurun_out/${TAG}_$1 python tools/prof_harness.py > gpurun_out/${TAG}_$1.log 2>&1
  echo "ncu $1 rc=$?"; tail -2 gpurun_out/${TAG}_$1.log
}
for k in ${KERNELS:-k1 splitk pair k2}; do
  case $k in
    k1) run k1 decode_attn_kernel 0 2 ;;
    splitk) run splitk tc_splitk_kernel 10 4 ;;
    pair) run pair tc_gemm_pair_kernel 0 4 ;;
    k2) run k2 chunk_attn_tc_kernel 0 2 ;;
  esac
done
