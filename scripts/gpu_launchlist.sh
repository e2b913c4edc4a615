#!/bin/bash
# ncu launch list (per-kernel device time) of one bench step + small driver
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-l}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
tail -2 gpurun_out/ncu_launch_$TAG.log
