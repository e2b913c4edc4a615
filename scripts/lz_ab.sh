#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/lanczos_probe.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C1 or C2 or C3" 2>&1 | tail -2
NUGPR_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lanczos -c 6 --csv python scripts/lanczos_probe.py 2>/dev/null | grep lanczos | awk -F'","' '{print $NF}' | head
timeout 300 python bench.py --steps 5 --no-cpu-baseline --prof-steps 1 > gpurun_out/blz.json 2>/dev/null
python - <<'PY'
import json
d=json.loads(open("gpurun_out/blz.json").read().strip().splitlines()[-1])
print(round(d["value"],1), d["config"]["phase_ms"], d["roofline"]["step_share"])
PY
