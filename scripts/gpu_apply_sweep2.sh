#!/bin/bash
# progressive-D x ring-slot sweep of the DMMA apply at C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "1 1024" "1 2048" "1 4096" "0 1024" "0 2048" "0 4096"; do
  set -- $spec
  NUGPR_APPLY_PROG=$1 NUGPR_APPLY_SLOT=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --prof-steps 2 > gpurun_out/sw2.json 2>/dev/null
  python - "$spec" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/sw2.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(f"prog/slot={sys.argv[1]:10s} value={d['value']:.1f} ms/step={d['ms_per_step']:.3f} apply_us={r['avg_launch_us']:.2f} frac={r['frac']:.3f}", flush=True)
PY
done
