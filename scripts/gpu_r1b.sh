#!/bin/bash
# Round-1 iteration: GPU tests, smoke, bench (no cpu baseline), launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-b}
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --no-cpu-baseline --eval-slots 1 > gpurun_out/bench1_$TAG.json 2>> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/bench1_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
