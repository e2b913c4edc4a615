"""Small driver for ncu captures: one C3 build + one evaluation per operator mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12128_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
ds = synth.make_config(cfg)
ctx = P.Context(0)
X = torch.tensor(ds.X, device="cuda"); y = torch.tensor(ds.y, device="cuda"); reps = torch.tensor(ds.reps, device="cuda")
b = P.build_blocks(ctx, X, ds.offsets, reps, ds.theta0)
l, s, a = ds.theta0
for th in [(l, s * 1.001, a), (l * 1.001, s, a), (l, s, a)]:
    P.mll(ctx, b, y, th, probe_seed=ds.meta["probe_seed"])
torch.cuda.synchronize()
print("done")
