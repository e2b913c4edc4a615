#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pyt_par.log 2>&1; tail -2 gpurun_out/pyt_par.log
for dbg in 0 1; do NUGPR_APPLY_DBG=$dbg timeout 120 python scripts/apply_micro.py C3; done
timeout 200 python scripts/apply_micro.py C5 2
NUGPR_APPLY_DBG=1 timeout 200 python scripts/apply_micro.py C5 2
