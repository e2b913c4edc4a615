#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2510_12128_b200 as P
ds = synth.make_config(sys.argv[1])
ctx = P.Context(0)
X = torch.tensor(ds.X, device="cuda"); y = torch.tensor(ds.y, device="cuda"); R = torch.tensor(ds.reps, device="cuda")
b = P.build_blocks(ctx, X, ds.offsets, R, ds.theta0)
l, s, a = ds.theta0
P.mll(ctx, b, y, (l, s * 1.001, a), probe_seed=1, replay=[1] * 9)
torch.cuda.synchronize()
PY
for dbg in 16 17; do
NUGPR_NO_GRAPH=1 NUGPR_APPLY_DBG=$dbg timeout 300 python /tmp/one.py C3 > gpurun_out/trace_C3.txt 2>&1
echo "== C3 staged dbg=$dbg"; python scripts/apply_trace.py gpurun_out/trace_C3.txt
done
