"""Print Lanczos iteration counts and lambda_0 accuracy at C1-C3 (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2510_12128_b200 as P
from oracle.structured import krep_and_M
ctx = P.Context(0)
for name in ["C1", "C2", "C3", "C5"]:
    ds = synth.make_config(name)
    b = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
    it, conv = b.lanczos_info("build")
    lam = b.export("scalars")[1]
    _, lam_ref, _ = krep_and_M("rbf", ds.reps, ds.theta0)
    th = (ds.theta0[0] * 1.001, ds.theta0[1], ds.theta0[2])
    rec = P.mll(ctx, b, ds.y, th, probe_seed=1)
    it2, conv2 = b.lanczos_info("eval")
    _, lam2, _ = krep_and_M("rbf", ds.reps, th)
    print(name, "build iters", it, conv, "rel err", abs(lam - lam_ref) / lam_ref, "| warm iters", it2, conv2,
          "rel err", abs(rec["lambda0"] - lam2) / lam2, flush=True)
    del b
