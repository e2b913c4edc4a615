#!/bin/bash
# A/B of the 4-CTA/SM DMMA apply (NW = 3, one cluster per CTA) against the 2-CTA/SM one at C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-as}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C3 or C2 or all_modes or f32 or graph or slots" > gpurun_out/pyt_as_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_as_$TAG.log; tail -3 gpurun_out/pyt_as_$TAG.log
for SM in 1 0; do
NUGPR_APPLY_SMALL=$SM timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_small$SM.json 2> gpurun_out/bench_${TAG}_small$SM.err
python - <<PY
import json; d = json.load(open("gpurun_out/bench_${TAG}_small$SM.json"))
r = d["roofline"]
print("small=$SM value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), "apply us", round(r["avg_launch_us"], 2), "frac", round(r["frac"], 3), "phase", d["config"]["phase_ms"])
PY
done
NUGPR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_mma -s 40 -c 1 -o gpurun_out/prof_apply_small_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_small_$TAG.log 2>&1; tail -1 gpurun_out/ncu_small_$TAG.log
