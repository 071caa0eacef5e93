#!/bin/bash
# A/B of a K1 launch knob on the C1 bench window: bash tools/k1_ab.sh VAR steps values...
VAR=$1; STEPS=$2; shift 2
mkdir -p gpurun_out
for m in "$@"; do
  env $VAR=$m timeout 600 python bench.py --steps $STEPS --warmup 5 --no-cpu-baseline > gpurun_out/k1ab_${VAR}_$m.json 2>/dev/null
  python - "$VAR" "$m" <<'PY'
import json, sys
j = json.loads(open(f"gpurun_out/k1ab_{sys.argv[1]}_{sys.argv[2]}.json").read().splitlines()[-1])
print(sys.argv[1], sys.argv[2], "req/s %.3f" % j["value"], "ms/step %.3f" % j["ms_per_step"],
      "K1 GB/s %.0f frac %.3f" % (j["roofline"]["achieved"], j["roofline"]["frac"]), "sm_mhz", j["clocks"]["sm_mhz"])
PY
done
