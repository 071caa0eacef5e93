#!/bin/bash
# Round-2 GPU session: parity tests, smoke, the C4 bench (both arms).
# Usage: gpurun --timeout 3000 -- 'bash tools/gpu_r2.sh TAG'
TAG=${1:-r2}
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/${TAG}_host.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
  tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200
fi
timeout 1200 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
  cat gpurun_out/${TAG}_ref.json; tail -3 gpurun_out/${TAG}_ref.err
fi
