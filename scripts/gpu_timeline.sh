#!/bin/bash
# numgrad timeline (per-eval start / pre-work / end) and the Cholesky phase trace at C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-tl}
NUGPR_TIMELINE=1 timeout 600 python - > gpurun_out/timeline_$TAG.log 2>&1 <<'PY'
import os, sys, time, torch, numpy as np
sys.path.insert(0, ".")
import synth, paper_2510_12128_b200 as P
ds = synth.make_config("C3")
ctx = P.Context(0)
dev = torch.device("cuda", 0)
Xd, rd, yd = torch.tensor(ds.X, device=dev), torch.tensor(ds.reps, device=dev), torch.tensor(ds.y, device=dev)
ws = torch.empty(P.workspace_size(ds.offsets, ds.n_c, ds.d, 7), dtype=torch.uint8, device=dev)
b = P.build_blocks(ctx, Xd, ds.offsets, rd, ds.theta0, workspace=ws, eval_slots=7)
for k in range(3):
    P.numgrad(ctx, b, yd, ds.theta0, probe_seed=203)
print("---- measured", flush=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
P.numgrad(ctx, b, yd, ds.theta0, probe_seed=203)
torch.cuda.synchronize()
print("numgrad host wall ms", 1e3 * (time.perf_counter() - t0))
PY
cat gpurun_out/timeline_$TAG.log | tail -12
NUGPR_CHOL_TRACE=1 timeout 300 python - > gpurun_out/cholphase_$TAG.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, ".")
import synth, paper_2510_12128_b200 as P
ds = synth.make_config("C3")
ctx = P.Context(0)
for k in range(2):
    b = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
    torch.cuda.synchronize()
    b.close()
PY
tail -8 gpurun_out/cholphase_$TAG.log
