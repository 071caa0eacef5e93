#!/bin/bash
# Quick GPU loop: parity tests (optionally a subset), smoke, short bench, iteration breakdown.
set -x
TAG=${1:-q}
TESTS=${TESTS:-tests}
mkdir -p gpurun_out
timeout 900 python -m pytest $TESTS -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/${TAG}_pytest.log
[ "${SKIP_BENCH:-0}" = 1 ] && exit 0
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
[ "${DIAG:-1}" = 1 ] && timeout 600 python tools/diag_iters.py 3000 300 > gpurun_out/${TAG}_iters.txt 2>&1; tail -10 gpurun_out/${TAG}_iters.txt
