#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f32" > gpurun_out/pyt_f32.log 2>&1; tail -15 gpurun_out/pyt_f32.log
NUGPR_APPLY_MMA=1 timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --blocks f32 > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; cat gpurun_out/bench_f32.json; tail -3 gpurun_out/bench_f32.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "50_epochs" > gpurun_out/pyt_train50.log 2>&1; tail -3 gpurun_out/pyt_train50.log
NUGPR_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "build_blocks_parity_C1 or mll_parity_C1_all_modes or numgrad_central_C1" > gpurun_out/san_memcheck.log 2>&1; tail -5 gpurun_out/san_memcheck.log
NUGPR_NO_GRAPH=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "mll_parity_C1_all_modes and baseline" > gpurun_out/san_racecheck.log 2>&1; tail -5 gpurun_out/san_racecheck.log
