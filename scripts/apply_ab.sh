#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "0 2" "1 2" "1 1"; do
  set -- $cfg
  NUGPR_APPLY_STAGE=$1 NUGPR_APPLY_PER=$2 timeout 200 python scripts/apply_micro.py C3 3
done
for cfg in "0 2" "1 2"; do
  set -- $cfg
  NUGPR_APPLY_STAGE=$1 NUGPR_APPLY_PER=$2 timeout 300 python bench.py --steps 5 --no-cpu-baseline --prof-steps 1 > gpurun_out/bab.json 2>/dev/null
  python - $1 <<'PY'
import json,sys
d=json.loads(open("gpurun_out/bab.json").read().strip().splitlines()[-1])
print("stage", sys.argv[1], round(d["value"],1), d["config"]["phase_ms"], round(d["roofline"]["avg_launch_us"],1))
PY
done
