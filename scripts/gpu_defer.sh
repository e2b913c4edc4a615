#!/bin/bash
# deferred build (H on its own stream, no host read-back) in nugpr_train: train parity + bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-df}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "train or scale or numgrad or shard" > gpurun_out/pyt_df_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_df_$TAG.log; tail -3 gpurun_out/pyt_df_$TAG.log
NUGPR_NO_GRAPH=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d = json.load(open('gpurun_out/bench_$TAG.json')); r = d['roofline']
print('value', round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value'], 1), 'apply us', round(r['avg_launch_us'], 2), 'frac', round(r['frac'], 3), 'phase', d['config']['phase_ms'])"
tail -2 gpurun_out/bench_$TAG.err
