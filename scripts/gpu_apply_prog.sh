#!/bin/bash
# A/B of the progressive-D DMMA apply (D_i rows arrive per chunk with the TMA stream) at C3, + parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ap}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C3 or C2 or all_modes or f32 or graph or slots or numgrad" > gpurun_out/pyt_ap_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_ap_$TAG.log; tail -3 gpurun_out/pyt_ap_$TAG.log
for PR in 1 0; do
NUGPR_APPLY_PROG=$PR timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_prog$PR.json 2> gpurun_out/bench_${TAG}_prog$PR.err
python - <<PY
import json; d = json.load(open("gpurun_out/bench_${TAG}_prog$PR.json"))
r = d["roofline"]
print("prog=$PR value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), "apply us", round(r["avg_launch_us"], 2), "frac", round(r["frac"], 3), "phase", d["config"]["phase_ms"])
PY
done
NUGPR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_mma -s 40 -c 1 -o gpurun_out/prof_apply_prog_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_prog_$TAG.log 2>&1; tail -1 gpurun_out/ncu_prog_$TAG.log
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; cut -c1-300 gpurun_out/bench_${TAG}_c5.json; python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c5.json')); print('C5 apply us', d['roofline']['avg_launch_us'], 'frac', d['roofline']['frac'])"
