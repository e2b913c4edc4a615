#!/bin/bash
# PAR-2 cluster sharding: shard tests (gloo world 2/3 on one GPU, NCCL world 1), then the regular
# parity suite subset that exercises the refactored finalisers, then sharded benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-par2}
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x -k "many_clusters" > gpurun_out/pyt_exact_$TAG.log 2>&1; tail -3 gpurun_out/pyt_exact_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/pyt_shard_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_shard_$TAG.log; tail -25 gpurun_out/pyt_shard_$TAG.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pyt_parity_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_parity_$TAG.log; tail -5 gpurun_out/pyt_parity_$TAG.log
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --shard clusters --no-cpu-baseline > gpurun_out/bench_c3_shard_$TAG.json 2> gpurun_out/bench_c3_shard_$TAG.err; cut -c1-600 gpurun_out/bench_c3_shard_$TAG.json; tail -3 gpurun_out/bench_c3_shard_$TAG.err
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --shard clusters --no-cpu-baseline > gpurun_out/bench_c5_shard_$TAG.json 2> gpurun_out/bench_c5_shard_$TAG.err; cut -c1-600 gpurun_out/bench_c5_shard_$TAG.json; tail -3 gpurun_out/bench_c5_shard_$TAG.err
