#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
NUGPR_DEBUG_SYNC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "build_blocks_parity or mll_parity_C1" > gpurun_out/debug.log 2>&1
echo "rc=$?" >> gpurun_out/debug.log
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -m5 -E "nugpr\]|Error|error" gpurun_out/debug.log; tail -3 gpurun_out/debug.log; tail -5 gpurun_out/pytest_gpu.log; head -20 gpurun_out/nvsmi.txt
