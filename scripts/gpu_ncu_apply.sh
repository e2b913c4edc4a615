#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-a}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_kernel -s 2 -c 1 -o gpurun_out/prof_apply_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_apply_$TAG.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/ncu_apply_$TAG.log; tail -2 gpurun_out/pytest_gpu_$TAG.log
