"""Per-evaluation latency probe (DESIGN §7 scaling model inputs).

    python tools/probe_evals.py [C3 ...]

For each config: the build time, Lanczos iteration counts (build and a lengthscale step), and
the device time of each of the 7 central-difference evaluations ALONE (graph mode, one slot,
median of 5, CUDA events on the context stream), plus the concurrent 7-evaluation numgrad.
"""
import json
import os
import statistics
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_12128_b200 as P  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=5):
    s = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    cfgs = sys.argv[1:] or ["C3"]
    ctx = P.Context(0)
    for cfg in cfgs:
        ds = synth.make_config(cfg)
        seed = ds.meta["probe_seed"]
        X = torch.tensor(ds.X, device="cuda")
        y = torch.tensor(ds.y, device="cuda")
        reps = torch.tensor(ds.reps, device="cuda")
        th0 = tuple(ds.theta0)
        res = {"config": cfg}
        b1 = P.build_blocks(ctx, X, ds.offsets, reps, th0, eval_slots=1)
        res["build_ms"] = timed(lambda: P.build_blocks(ctx, X, ds.offsets, reps, th0, eval_slots=1).close())
        res["lanczos_build"] = b1.lanczos_info("build")
        pts = [th0]
        for i in range(3):
            for sg in (1, -1):
                q = list(th0)
                q[i] = th0[i] + sg * 1e-3 * th0[i]
                pts.append(tuple(q))
        names = ["base", "lam+", "lam-", "noise+", "noise-", "scale+", "scale-"]
        ev = {}
        for nm, p in zip(names, pts):
            P.mll(ctx, b1, y, p, probe_seed=seed)
            ev[nm] = timed(lambda p=p: P.mll(ctx, b1, y, p, probe_seed=seed))
            if nm == "lam+":
                res["lanczos_lam"] = b1.lanczos_info("eval")
            r = P.mll(ctx, b1, y, p, probe_seed=seed)
            ev[nm + "_iters"] = [r["iters_y"], r["iters_q_max"]]
        res["eval_ms_alone"] = ev
        b7 = P.build_blocks(ctx, X, ds.offsets, reps, th0, eval_slots=7)
        P.numgrad(ctx, b7, y, th0, probe_seed=seed)
        res["numgrad7_concurrent_ms"] = timed(lambda: P.numgrad(ctx, b7, y, th0, probe_seed=seed))
        res["numgrad7_serial_ms"] = timed(lambda: P.numgrad(ctx, b1, y, th0, probe_seed=seed))
        print(json.dumps(res), flush=True)
        b1.close()
        b7.close()


if __name__ == "__main__":
    main()
