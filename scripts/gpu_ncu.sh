#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-n}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_kernel -s 2 -c 1 -o gpurun_out/prof_apply_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_apply_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos -s 0 -c 1 -o gpurun_out/prof_lanczos_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_lanczos_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_trtri -s 0 -c 1 -o gpurun_out/prof_chol_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_chol_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_blocks -s 0 -c 3 -o gpurun_out/prof_gemm_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_gemm_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:update_kernel -s 3 -c 1 -o gpurun_out/prof_update_$TAG python scripts/prof_driver.py C3 > gpurun_out/ncu_update_$TAG.log 2>&1
ls -la gpurun_out/*$TAG*; tail -2 gpurun_out/ncu_apply_$TAG.log
