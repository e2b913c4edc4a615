#!/bin/bash
# grid balance / CTAs-per-SM sweep of the DMMA apply at C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "2 1" "2 0" "1 0" "1 1"; do
  set -- $spec
  NUGPR_APPLY_PER=$1 NUGPR_APPLY_BAL=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --prof-steps 2 > gpurun_out/sw3.json 2>/dev/null
  python - "$spec" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/sw3.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(f"per/bal={sys.argv[1]:6s} value={d['value']:.1f} ms/step={d['ms_per_step']:.3f} apply_us={r['avg_launch_us']:.2f} frac={r['frac']:.3f}", flush=True)
PY
done
