#!/bin/bash
# One GPU session: parity tests, smoke, bench line, launch list, ncu capture of K1.
# Usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  -c 1500 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "ncu list rc=$?"
BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:decode_attn_kernel -c 2 -o gpurun_out/${TAG}_k1 \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_k1_bench.log 2>&1; echo "ncu k1 rc=$?"
BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:tc_gemm -c 4 -o gpurun_out/${TAG}_k3 \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_k3_bench.log 2>&1; echo "ncu k3 rc=$?"
ls -la gpurun_out
