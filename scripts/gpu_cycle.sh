#!/bin/bash
# One dev cycle: GPU tests, bench (no cpu baseline), ncu of the apply kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-c}
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-apply_kernel} -s ${KSKIP:-2} -c 1 -o gpurun_out/prof_k_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_k_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err; tail -1 gpurun_out/ncu_k_$TAG.log
