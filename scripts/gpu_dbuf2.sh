#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for m in 2 1; do NUGPR_APPLY_DBUF=$m timeout 120 python scripts/apply_micro.py C3 2>&1 | grep -v Warn; done
for m in 2 1; do
NUGPR_APPLY_DBUF=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_db$m.json 2> gpurun_out/bench_db$m.err
python -c "
import json; d = json.load(open('gpurun_out/bench_db$m.json')); r = d['roofline']
print('dbuf=$m value', round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value'], 1), 'apply us', round(r['avg_launch_us'], 2), 'frac', round(r['frac'], 3), 'phase', d['config']['phase_ms'])"
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big.py tests/test_gpu_shard.py -q -x -k "C3 or C2 or all_modes or f32 or graph or slots or uneven or mbcg or nccl or train" > gpurun_out/pyt_db.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_db.log; tail -3 gpurun_out/pyt_db.log
