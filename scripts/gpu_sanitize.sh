#!/bin/bash
# compute-sanitizer memcheck / racecheck over small parity cases of the final code (direct launches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NUGPR_NO_GRAPH=1 timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "build_blocks_parity_C1 or mll_parity_C1_all_modes or numgrad_central_C1 or uneven_ragged" > gpurun_out/san_memcheck_r01l.log 2>&1; tail -4 gpurun_out/san_memcheck_r01l.log
NUGPR_NO_GRAPH=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "mll_parity_C1_all_modes and noise" > gpurun_out/san_racecheck_r01l.log 2>&1; tail -4 gpurun_out/san_racecheck_r01l.log
