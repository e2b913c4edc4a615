"""Apply-kernel micro timing: noise-mode MLL evaluations at a config in the event-profiled path;
prints the average apply-with-B launch time and the achieved algorithmic GB/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2510_12128_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps_n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ds = synth.make_config(cfg)
ctx = P.Context(0)
X = torch.tensor(ds.X, device="cuda"); y = torch.tensor(ds.y, device="cuda"); R = torch.tensor(ds.reps, device="cuda")
b = P.build_blocks(ctx, X, ds.offsets, R, ds.theta0)
l, s, a = ds.theta0
th = (l, s * 1.001, a)
P.mll(ctx, b, y, th, probe_seed=ds.meta["probe_seed"], replay=[6] * 9)
ctx.set_profiling(True)
for _ in range(reps_n):
    P.mll(ctx, b, y, th, probe_seed=ds.meta["probe_seed"], replay=[6] * 9)
ms, by, n = ctx.profile()["apply_B"]
print(f"{cfg} dbg={os.environ.get('NUGPR_APPLY_DBG','0')} per={os.environ.get('NUGPR_APPLY_PER','2')} "
      f"slot={os.environ.get('NUGPR_APPLY_SLOT','4096')}: apply_B {1e3*ms/n:.2f} us/launch, {by/ms/1e6:.0f} GB/s ({n} launches)")
