#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-b}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos -s 1 -c 1 -o gpurun_out/prof_lz_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_lz_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_trtri -s 0 -c 1 -o gpurun_out/prof_ch_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_ch_$TAG.log 2>&1
timeout 600 python scripts/lanczos_probe.py > gpurun_out/lanczos_$TAG.log 2>&1
tail -1 gpurun_out/ncu_lz_$TAG.log; tail -1 gpurun_out/ncu_ch_$TAG.log; cat gpurun_out/lanczos_$TAG.log
