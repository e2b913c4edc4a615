#!/bin/bash
# NEXT-2 exact evaluator + NEXT-4 mBCG parity, then benches of the estimator / storage variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > gpurun_out/pyt_exact.log 2>&1; tail -15 gpurun_out/pyt_exact.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mbcg" > gpurun_out/pyt_mbcg.log 2>&1; tail -15 gpurun_out/pyt_mbcg.log
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --logdet mbcg --no-cpu-baseline > gpurun_out/bench_mbcg.json 2> gpurun_out/bench_mbcg.err; cat gpurun_out/bench_mbcg.json; tail -3 gpurun_out/bench_mbcg.err
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --blocks f32 --no-cpu-baseline > gpurun_out/bench_f32b.json 2> gpurun_out/bench_f32b.err; cat gpurun_out/bench_f32b.json; tail -3 gpurun_out/bench_f32b.err
timeout 1200 python -m pytest tests/test_gpu_big.py -q -x -k "C5" > gpurun_out/pyt_c5.log 2>&1; tail -5 gpurun_out/pyt_c5.log
