#!/bin/bash
# Round-2 evidence pass: bench C3 (solo evaluation latencies), C5 replicated vs cluster-sharded
# (in-library NCCL), ncu --set full of one packed apply (DRAM traffic), sanitizers on C1/C2 cases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=r02d
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_C3.json 2> gpurun_out/${T}_bench_C3.err; cut -c1-200 gpurun_out/${T}_bench_C3.json
timeout 900 python bench.py --config C5 --no-cpu-baseline --train-epochs 0 --shard clusters > gpurun_out/${T}_bench_C5_shard.json 2> gpurun_out/${T}_bench_C5_shard.err; cut -c1-200 gpurun_out/${T}_bench_C5_shard.json; tail -2 gpurun_out/${T}_bench_C5_shard.err
TAG=$T CFG=C3 SKIP=40 NLINES=10 tools/ncu_apply.sh > /dev/null 2>&1; head -c 600 gpurun_out/${T}_ncu_C3_apply_packed.jsonl; echo
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
     -k "C1_all_modes or uneven or numgrad_central_C1 or graph_mode_equals" > gpurun_out/${T}_sanitizer_${tool}_C1.log 2>&1
  echo "$tool: $(tail -n 1 gpurun_out/${T}_sanitizer_${tool}_C1.log)"
done
timeout 900 compute-sanitizer --tool racecheck --target-processes all python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
   -k "C2 and not f32 and not train and not mbcg" > gpurun_out/${T}_sanitizer_racecheck_C2.log 2>&1
echo "racecheck C2: $(grep -c 'Race reported' gpurun_out/${T}_sanitizer_racecheck_C2.log) race reports; $(tail -n 1 gpurun_out/${T}_sanitizer_racecheck_C2.log)"
