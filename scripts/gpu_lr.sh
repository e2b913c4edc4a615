#!/bin/bash
# lowrank with two T rows per warp + deduplicated epilogue loads: bench + launch list + parity subset
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lr.json 2> gpurun_out/bench_lr.err
python -c "
import json; d = json.load(open('gpurun_out/bench_lr.json')); r = d['roofline']
print('value', round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value'], 1), 'apply us', round(r['avg_launch_us'], 2), 'frac', round(r['frac'], 3), 'phase', d['config']['phase_ms'], r['step_share'])"
NUGPR_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_lr.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_launch_lr.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_lr.csv 2>/dev/null | head -6
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "C3 or C2 or all_modes or graph or slots or uneven or nccl" > gpurun_out/pyt_lr.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_lr.log; tail -3 gpurun_out/pyt_lr.log
