#!/bin/bash
# bench lines of the other configs / variants on the final code
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --blocks f32 --no-cpu-baseline > gpurun_out/bench_f32_r01l.json 2>/dev/null
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_r01l.json 2>/dev/null
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r01l.json 2>/dev/null
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_r01l.json 2>/dev/null
for f in f32 c4 c5 c2; do python -c "
import json; d = json.load(open('gpurun_out/bench_${f}_r01l.json')); r = d['roofline']
print('$f', d['config']['workload'][:12], 'value', round(d['value'], 2), 'ms/step', round(d['ms_per_step'], 3), 'apply us', round(r['avg_launch_us'] or 0, 2), 'frac', round(r['frac'] or 0, 3), 'peak GB', round(d['config']['peak_hbm_gb'], 2))"; done
