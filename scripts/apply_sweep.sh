#!/bin/bash
# Sweep apply-kernel launch plans (env knobs of plan_apply) on the bench config.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C3}
for spec in "2 4096 0" "2 4096 1" "2 2048 1" "2 1024 1" "1 4096 1" "1 2048 1" "1 8192 1"; do
  set -- $spec
  NUGPR_APPLY_PER=$1 NUGPR_APPLY_SLOT=$2 NUGPR_APPLY_BAL=$3 timeout 300 python bench.py --config $CFG --steps 5 --no-cpu-baseline --prof-steps 2 > gpurun_out/sw.json 2>/dev/null
  python - "$spec" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/sw.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(f"per/slot/bal={sys.argv[1]:12s} value={d['value']:.1f} ms/step={d['ms_per_step']:.2f} apply_us={r['avg_launch_us']:.2f} frac={r['frac']:.3f}")
PY
done
