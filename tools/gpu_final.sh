#!/bin/bash
# Round-end rehearsal on one B200: the whole GPU suite, smoke, the default bench (C4, both arms),
# the C0 line (CPU path over the whole trace) and the CPU depth check.
TAG=${1:-r2final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log; grep -E "^FAILED" gpurun_out/${TAG}_pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-150
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json | cut -c1-400
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 --validate-depth > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
cat gpurun_out/${TAG}_ref.json | cut -c1-400
timeout 900 python bench.py --config C0 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_c0.json 2> gpurun_out/${TAG}_c0.err; echo "c0 rc=$?"
timeout 900 python bench.py --impl reference --config C0 --full-trace --steps 20 --warmup 5 > gpurun_out/${TAG}_c0ref.json 2> gpurun_out/${TAG}_c0ref.err; echo "c0ref rc=$?"
timeout 900 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_c1.json 2> gpurun_out/${TAG}_c1.err; echo "c1 rc=$?"
for f in c0 c0ref c1; do python -c "import json; d=json.load(open('gpurun_out/${TAG}_$f.json')); print('$f', d['value'], d['ms_per_step'])"; done
