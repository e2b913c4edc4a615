#!/bin/bash
# Build-phase trace at C3 (host wall clock per phase) and the bench with one train call for K epochs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-bt}
NUGPR_BUILD_TRACE=1 timeout 600 python - > gpurun_out/build_trace_$TAG.log 2>&1 <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, ".")
import synth, paper_2510_12128_b200 as P
ds = synth.make_config("C3")
ctx = P.Context(0)
dev = torch.device("cuda", 0)
Xd, rd, yd = torch.tensor(ds.X, device=dev), torch.tensor(ds.reps, device=dev), torch.tensor(ds.y, device=dev)
ws = torch.empty(P.workspace_size(ds.offsets, ds.n_c, ds.d, 7), dtype=torch.uint8, device=dev)
for k in range(4):
    b = P.build_blocks(ctx, Xd, ds.offsets, rd, ds.theta0, workspace=ws, eval_slots=7)
    b.close()
st = np.zeros(10); st[:3] = ds.theta0
P.train(ctx, Xd, ds.offsets, rd, yd, None, epochs=3, adam_state=st, workspace=ws, probe_seed=203)
PY
cat gpurun_out/build_trace_$TAG.log | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cut -c1-900 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
