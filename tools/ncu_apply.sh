#!/bin/bash
# ncu --set full capture of one packed apply with a block term at a config (direct launches).
#   TAG=name CFG=C3 KREGEX=apply_packed SKIP=40 tools/ncu_apply.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}; CFG=${CFG:-C3}; KREGEX=${KREGEX:-apply_packed}; SKIP=${SKIP:-40}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $SKIP -c 1 \
  -f -o gpurun_out/${TAG}_ncu_${CFG}_${KREGEX} python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 1 \
  --train-epochs 0 --direct > gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.log 2>&1
tail -2 gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.log
python tools/ncu_summary.py gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.ncu-rep > gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.jsonl
cut -c1-1500 gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.jsonl; python tools/ncu_lines.py gpurun_out/${TAG}_ncu_${CFG}_${KREGEX}.ncu-rep ${NLINES:-20}
