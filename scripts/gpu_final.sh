#!/bin/bash
# Round-end pass: the whole GPU suite (incl. PAR-2 C5 world-4), smoke, default bench + C5 sharded bench,
# launch list and one full ncu capture of the dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-fin}
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cut -c1-300 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; cut -c1-300 gpurun_out/bench_ref_$TAG.json
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --shard clusters --no-cpu-baseline > gpurun_out/bench_c5s_$TAG.json 2> gpurun_out/bench_c5s_$TAG.err; cut -c1-200 gpurun_out/bench_c5s_$TAG.json
NUGPR_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
NUGPR_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_mma -s 40 -c 1 -o gpurun_out/prof_apply_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1; tail -1 gpurun_out/ncu_full_$TAG.log
