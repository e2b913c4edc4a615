"""Per-CTA timeline of ONE packed apply launch (diagnostics build, libnugpr_trace.so).

    python -m paper_2510_12128_b200.build --trace          # here (cross-compiles)
    python tools/apply_trace.py [C3|C5|C2] [launch_index] [mode]   # on the GPU box

Runs one MLL evaluation with direct launches (noise step by default: a block term in every
apply) and records globaltimer stamps of the `launch_index`-th packed apply (0-based; per CG
iteration the fused first apply then the second).  Prints per-CTA phase times relative to the
earliest CTA start and a summary.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mode = sys.argv[3] if len(sys.argv) > 3 else "noise"
os.environ["NUGPR_TRACE_AT"] = str(idx)

import torch  # noqa: E402

import paper_2510_12128_b200 as P  # noqa: E402
from paper_2510_12128_b200 import _native  # noqa: E402
import synth  # noqa: E402

_native.LIB_PATH = os.path.join(ROOT, "paper_2510_12128_b200", "libnugpr_trace.so")
lib = _native.lib()
ds = synth.make_config(cfg)
ctx = P.Context(0)
ctx.set_option("graphs", False)
bl = P.build_blocks(ctx, torch.tensor(ds.X, device="cuda"), ds.offsets, torch.tensor(ds.reps, device="cuda"),
                    ds.theta0)
y = torch.tensor(ds.y, device="cuda")
l, s, a = ds.theta0
th = {"noise": (l, s * 1.001, a), "scale": (l, s, a * 1.001), "generic": (l * 1.001, s, a)}[mode]
rec = P.mll(ctx, bl, y, th, probe_seed=ds.meta["probe_seed"])
torch.cuda.synchronize()
buf = (C.c_ulonglong * (148 * 64))()
fn = lib.nugpr_debug_apply_trace
fn.argtypes = [C.c_void_p]
assert fn(buf) == 0
T = np.frombuffer(buf, dtype=np.uint64).reshape(148, 64).astype(np.int64)
t0 = T[:, 0].min()
us = lambda v: (v - t0) / 1000.0 if v > 0 else float("nan")  # noqa: E731
print(f"{cfg} {mode} apply #{idx}: iters_y={rec['iters_y']} iters_q={rec['iters_q_max']}")
ends = []
for b in range(148):
    r = T[b]
    nseg = int(r[46])
    ends.append(us(r[45]))
    line = [f"cta {b:3d} nseg {nseg:2d} start {us(r[0]):6.1f} M' {us(r[1]):6.1f} S {us(r[3]):6.1f} lr {us(r[28]):6.1f} prod_end {us(r[2]):6.1f}"]
    for q in range(min(nseg, 8)):
        line.append(f" | q{q} mma {us(r[4+q]):6.1f}-{us(r[12+q]):6.1f} free {us(r[20+q]):6.1f} epi {us(r[29+q]):6.1f}-{us(r[37+q]):6.1f}")
    line.append(f" | end {us(r[45]):6.1f}")
    print("".join(line))
e = np.array(ends)
wt, ct = T[:, 48].astype(float), T[:, 49].astype(float)
print(f"MMA warp 0 cycles: chunk waits median {np.median(wt):.0f}, block compute median {np.median(ct):.0f} "
      f"(sum median {np.median(wt + ct):.0f})")
mhz = T[:, 47].astype(float) / np.maximum(1e-9, (T[:, 45] - T[:, 0]).astype(float)) * 1e3
print(f"effective SM clock over the kernel: median {np.median(mhz):.0f} MHz")
pw = T[:, 56:64].astype(float)
print(f"MMA warps (blocks + chunk waits) cycles: per-CTA min over warps median {np.median(pw.min(1)):.0f}, "
      f"max over warps median {np.median(pw.max(1)):.0f}; per warp median {np.median(pw, 0).astype(int).tolist()}")
for k, nm in [(50, "dready waits"), (51, "accfree waits"), (52, "esplit + tail"), (53, "piece intervals")]:
    print(f"  warp 0 {nm:16s}: median {np.median(T[:, k].astype(float)):.0f} cycles")
print(f"kernel end: min {np.nanmin(e):.1f} median {np.nanmedian(e):.1f} max {np.nanmax(e):.1f} us")
first_mma = np.array([us(T[b][4]) for b in range(148)])
print(f"first MMA piece start: median {np.nanmedian(first_mma):.1f} max {np.nanmax(first_mma):.1f}")
for k, nm in [(1, "M' rows staged"), (3, "S rows staged")]:
    v = np.array([us(T[b][k]) for b in range(148)])
    print(f"{nm}: median {np.nanmedian(v):.1f} max {np.nanmax(v):.1f}")
lr = np.array([us(T[b][28]) for b in range(148)])
print(f"low-rank rows done: median {np.nanmedian(lr):.1f} max {np.nanmax(lr):.1f}")
