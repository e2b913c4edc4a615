#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pyt_par.log 2>&1; tail -2 gpurun_out/pyt_par.log
for cfg in C3 C5; do
  for dbg in 0 4 1 3; do
  NUGPR_APPLY_DBG=$dbg timeout 200 python scripts/apply_micro.py $cfg 2
  done
done
