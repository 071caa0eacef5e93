#!/bin/bash
# C4 profiling session (1 GPU): launch list of the bench's timed windows (ncu,
# one metric, serialised and cold: kernel SHARES, not absolute times) and the
# per-iteration phase breakdown.
# Usage: gpurun --timeout 2400 -- 'bash tools/gpu_prof_c4.sh TAG'
TAG=${1:-r2}
CFG=${CFG:-C4}
mkdir -p gpurun_out
BENCH_PROFILE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  -c 20000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --config $CFG --steps ${STEPS:-8} --warmup 3 --windows ${WINDOWS:-4} --no-cpu-baseline \
  > gpurun_out/${TAG}_launches_bench.log 2>&1; echo "ncu list rc=$?"
tail -2 gpurun_out/${TAG}_launches_bench.log | cut -c1-300
python tools/launch_shares.py gpurun_out/${TAG}_launches.csv ${STEPS:-8} > gpurun_out/${TAG}_launch_shares.txt
cat gpurun_out/${TAG}_launch_shares.txt | head -30
gzip -f gpurun_out/${TAG}_launches.csv
