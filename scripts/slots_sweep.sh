#!/bin/bash
cd "$(dirname "$0")/.."
for sl in 2 3 4 7; do
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python bench.py --steps 5 --no-cpu-baseline --prof-steps 1 --eval-slots $sl > gpurun_out/bsl.json 2>/dev/null
python - $sl <<'PY'
import json,sys
d=json.loads(open("gpurun_out/bsl.json").read().strip().splitlines()[-1])
print("slots", sys.argv[1], round(d["value"],1), d["config"]["phase_ms"])
PY
done
