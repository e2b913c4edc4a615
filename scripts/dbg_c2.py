import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2510_12128_b200 as P
ds = synth.make_config("C2")
ctx = P.Context(0)
b = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
r = P.mll(ctx, b, ds.y, ds.theta0, probe_seed=202)
print(r["L"], r["iters_y"])
