#!/bin/bash
# compute-sanitizer over the hot path: memcheck / racecheck /
# synccheck / initcheck on smoke (tiny model: prefill chunks, decode rows,
# K1/K2/K3/K4/K8), and memcheck + synccheck on the swap and chunk-attention tests.
# Usage: gpurun --timeout 3600 -- 'bash tools/gpu_sanitize.sh TAG'
TAG=${1:-r2}
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20 --error-exitcode 99"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/${TAG}_san_smoke_${tool}.log 2>&1; echo "smoke $tool rc=$?"
  tail -4 gpurun_out/${TAG}_san_smoke_${tool}.log | cut -c1-240
done
for tool in memcheck synccheck racecheck; do
  timeout 1500 $CS --tool $tool python -m pytest -q -p no:cacheprovider -m gpu \
    tests/test_gpu_swap.py tests/test_gpu_chunk_attention.py tests/test_gpu_async.py::test_async_path_matches_sync_dynamic \
    > gpurun_out/${TAG}_san_tests_${tool}.log 2>&1; echo "tests $tool rc=$?"
  tail -4 gpurun_out/${TAG}_san_tests_${tool}.log | cut -c1-240
done
