#!/bin/bash
# memcheck / racecheck where the double-buffered D_i prefetch (cp.async) is active (ld = 200: C2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NUGPR_NO_GRAPH=1 timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "mll_parity_C2" > gpurun_out/san_memcheck_C2_r01l.log 2>&1; tail -4 gpurun_out/san_memcheck_C2_r01l.log
NUGPR_NO_GRAPH=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "mll_parity_C2 and noise" > gpurun_out/san_racecheck_C2_r01l.log 2>&1; tail -4 gpurun_out/san_racecheck_C2_r01l.log
