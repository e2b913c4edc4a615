#!/bin/bash
# Round pass: full GPU tests, smoke, benches (C3 default, C4), launch list and one full ncu capture
# of the dominant kernel (graphs off for the ncu runs: ncu cannot profile conditional-graph nodes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r}
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > gpurun_out/bench_c4_$TAG.json 2>> gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
NUGPR_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
NUGPR_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_mma -s 40 -c 1 -o gpurun_out/prof_apply_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -1 gpurun_out/smoke_$TAG.log; cat gpurun_out/bench_$TAG.json | cut -c1-400; cat gpurun_out/bench_c4_$TAG.json | cut -c1-400; tail -3 gpurun_out/bench_$TAG.err; tail -1 gpurun_out/ncu_full_$TAG.log
