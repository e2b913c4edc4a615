#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for dbg in 0 1 2 3; do NUGPR_APPLY_DBG=$dbg timeout 120 python scripts/apply_micro.py C3; done
for slot in 8192 16384; do NUGPR_APPLY_SLOT=$slot NUGPR_APPLY_PER=1 timeout 120 python scripts/apply_micro.py C3; done
NUGPR_APPLY_DBG=3 NUGPR_APPLY_PER=1 NUGPR_APPLY_SLOT=16384 timeout 120 python scripts/apply_micro.py C3
timeout 200 python scripts/apply_micro.py C5 2
NUGPR_APPLY_DBG=1 timeout 200 python scripts/apply_micro.py C5 2
