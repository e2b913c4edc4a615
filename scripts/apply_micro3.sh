#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NUGPR_DEBUG_SYNC=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pyt_par.log 2>&1; tail -5 gpurun_out/pyt_par.log
for col in 1 0; do
  NUGPR_APPLY_COL=$col timeout 200 python scripts/apply_micro.py C3 3
  NUGPR_APPLY_COL=$col NUGPR_APPLY_DBG=1 timeout 200 python scripts/apply_micro.py C3 3
done
timeout 200 python scripts/apply_micro.py C2 3
