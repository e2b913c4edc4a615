#!/bin/bash
# where the C3 apply's time goes: dbg 1 = no math, 2 = no epilogue, 64 = no D_i load, 32 = no L2 prefetch
cd "$(dirname "$0")/.."
for dbg in 0 1 3 64 67 99; do NUGPR_APPLY_DBG=$dbg timeout 120 python scripts/apply_micro.py C3; done
for dbg in 0 3; do NUGPR_APPLY_PROG=1 NUGPR_APPLY_DBG=$dbg timeout 120 python scripts/apply_micro.py C3; done
NUGPR_APPLY_DBG=67 timeout 200 python scripts/apply_micro.py C5 2
