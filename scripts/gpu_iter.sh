#!/bin/bash
# Iteration pass: lanczos probe, GPU tests, bench (no cpu baseline).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 600 python scripts/lanczos_probe.py > gpurun_out/lanczos_$TAG.log 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/lanczos_$TAG.log | tail -8; tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
