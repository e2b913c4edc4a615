#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NUGPR_CHOL_SMEM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C1 or C2 or jitter or ragged or single" > gpurun_out/pyt_chol.log 2>&1; tail -2 gpurun_out/pyt_chol.log
for v in 0 1; do
NUGPR_CHOL_SMEM=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline --prof-steps 1 > gpurun_out/bchol.json 2>/dev/null
python - $v <<'PY'
import json,sys
d=json.loads(open("gpurun_out/bchol.json").read().strip().splitlines()[-1])
print("smem" if sys.argv[1]=="1" else "global", round(d["value"],1), d["config"]["phase_ms"], d["roofline"]["step_share"]["chol"])
PY
done
