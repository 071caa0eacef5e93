#!/bin/bash
# Profiling session (1 GPU): per-iteration breakdown, host-link peak, launch list
# of a 20-iteration window, and ncu --set full captures of the hot kernels.
# The ncu captures shrink the KV pool (--gpu-blocks) so ncu can save/restore
# device memory between kernel replays; the window only uses ~60 GB of KV.
set -x
TAG=${1:-r1}
KERNELS=${KERNELS:-"decode_attn_kernel tc_gemm_kernel tc_skinny_kernel chunk_attn_kernel"}
mkdir -p gpurun_out
if [ "${SKIP_DIAG:-0}" != 1 ]; then
timeout 600 python tools/diag_iters.py 3000 300 > gpurun_out/${TAG}_iters.txt 2>&1; echo "iters rc=$?"
cat gpurun_out/${TAG}_iters.txt | tail -12
timeout 300 python tools/diag_link.py > gpurun_out/${TAG}_link.txt 2>&1; cat gpurun_out/${TAG}_link.txt
BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  -c 8000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --gpu-blocks 10000 > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "ncu list rc=$?"
fi
for k in $KERNELS; do
BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:$k -c ${NCU_COUNT:-3} -o gpurun_out/${TAG}_$k \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline --gpu-blocks 10000 > gpurun_out/${TAG}_${k}_ncu.log 2>&1; echo "ncu $k rc=$?"
tail -3 gpurun_out/${TAG}_${k}_ncu.log
done
ls -la gpurun_out
