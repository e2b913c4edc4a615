import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2510_12128_b200 as P
ds = synth.make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = P.Context(0)
X = torch.tensor(ds.X, device="cuda"); R = torch.tensor(ds.reps, device="cuda")
for _ in range(4):
    b = P.build_blocks(ctx, X, ds.offsets, R, ds.theta0)
    torch.cuda.synchronize()
    print("----", flush=True)
