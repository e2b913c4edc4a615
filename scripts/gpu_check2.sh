#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-c2}
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x -k variants > gpurun_out/pyt_var_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_var_$TAG.log; tail -15 gpurun_out/pyt_var_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big.py -q -x -k "lam or generic or all_modes or C4 or numgrad or slq" > gpurun_out/pyt_g_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_g_$TAG.log; tail -3 gpurun_out/pyt_g_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d = json.load(open('gpurun_out/bench_$TAG.json')); r = d['roofline']
print('value', round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value'], 1), 'apply us', round(r['avg_launch_us'], 2), 'frac', round(r['frac'], 3), 'phase', d['config']['phase_ms'], r['step_share'])"
NUGPR_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv | head -12
