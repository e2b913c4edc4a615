import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2510_12128_b200 as P
ds = synth.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx = P.Context(0)
X = torch.tensor(ds.X, device="cuda"); y = torch.tensor(ds.y, device="cuda"); R = torch.tensor(ds.reps, device="cuda")
b = P.build_blocks(ctx, X, ds.offsets, R, ds.theta0, eval_slots=7)
for it in range(3):
    P.numgrad(ctx, b, y, ds.theta0, probe_seed=ds.meta["probe_seed"])
    torch.cuda.synchronize()
    print("----", file=sys.stderr, flush=True)
