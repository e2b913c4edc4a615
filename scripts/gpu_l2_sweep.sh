#!/bin/bash
# L2 evict_last share of H in the apply's TMA stream, C3 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for f in 0 0.3 0.5 0.7 1.0; do
  NUGPR_L2_FRAC=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --prof-steps 2 > gpurun_out/l2.json 2>/dev/null
  python - "$f" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/l2.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(f"l2frac={sys.argv[1]:5s} value={d['value']:.1f} ms/step={d['ms_per_step']:.3f} apply_us={r['avg_launch_us']:.2f} numgrad_ms={d['config']['phase_ms'].get('numgrad_ms',0):.3f}", flush=True)
PY
done
