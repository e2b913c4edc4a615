#!/bin/bash
# Full GPU pass: smoke, the whole -m gpu suite, the default bench line, the ncu launch list of the
# same bench command, and the C4/C5 bench lines.   TAG=r02a tools/gpu_pass.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
if [ -z "$NOTESTS" ]; then
timeout ${PYT_TIMEOUT:-1800} python -m pytest tests -q -m gpu ${PYT_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1
tail -${PYT_TAIL:-8} gpurun_out/${TAG}_pytest.log
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cut -c1-400 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --direct --train-epochs 0 \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches_C3.csv > gpurun_out/${TAG}_launches_C3.txt 2>&1; head -25 gpurun_out/${TAG}_launches_C3.txt
for C in C4 C5 C2; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --train-epochs 0 > gpurun_out/${TAG}_bench_$C.json 2> gpurun_out/${TAG}_bench_$C.err
  cut -c1-300 gpurun_out/${TAG}_bench_$C.json; tail -2 gpurun_out/${TAG}_bench_$C.err
done
