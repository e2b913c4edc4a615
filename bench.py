"""Benchmark of the nuGPR training hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

A "step" is one pass of the whole hot path (every row of SURVEY §8(a) except the one-off
clustering A0): one epoch of Algorithm 1 at config C3 (n=100,000, d=8,
n_c=500 clusters of 200, RBF, m=8 probes): build the preconditioner at theta (A1), the 2p+1 = 7
perturbed MLL evaluations of the central-difference gradient (A2-A8), Adam (A9).
value = MLL+num-grad evaluations per second (7 per step) over all ranks; PAR-1 shards the 7
evaluations of a step across ranks (strong scaling: the work per step is fixed).

--impl reference times the FP64 CPU oracle (oracle/, the only other place this script runs it)
on the same config and metric, each step a bounded sample (one of the 7 evaluations in turn,
plus the build every 7th step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# the 7 concurrent evaluation streams (+ side streams) need more hardware work queues than the
# default 8, or unrelated streams alias onto one queue and serialise; set before CUDA starts
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "MLL+num-grad evals/sec (n=100k, C3)"
UNIT = "evals/s"
CONFIG_DESC = {
    "C1": "n=1000 d=2 n_c=10 b=100 RBF m=8",
    "C2": "n=20000 d=8 n_c=100 b=200 RBF m=8",
    "C3": "n=100000 d=8 n_c=500 b=200 RBF m=8",
    "C4": "n=32000 (+8000 test) d=8 n_c=20 uneven k-means clusters, Matern-5/2, m=8",
    "C5": "n=1000000 d=4 n_c=2000 b=500 RBF m=8",
}


def load_config(name, P=None, ctx=None):
    """Dataset of a BASELINE config.  C4 (G-REAL) is clustered by row A0 first: on the GPU
    through the library (nugpr_cluster) for our arm, by the oracle's k-means for the reference
    arm (the two are bit-identical, tests/test_gpu_cluster.py); theta0 per the G-REAL recipe
    (median intra-cluster distance, 0.16, Var(y))."""
    if name != "C4":
        return synth.make_config(name)
    g = synth.g_real(N=40000, d=8, seed=104)
    if P is not None:
        r = P.cluster(ctx, g["X"], 20, y=g["y"], seed=104, rep_mode="centroid")
        X, y, off, reps = (r["X_sorted"].cpu().numpy(), r["y_sorted"].cpu().numpy(), r["offsets"],
                           r["reps"].cpu().numpy())
    else:
        from oracle import kmeans as KM
        km = KM.kmeans(g["X"], 20, seed=104, rep_mode=KM.CENTROID)
        X, y, off, reps = g["X"][km["perm"]], g["y"][km["perm"]], km["offsets"], km["reps"]
    rng = np.random.default_rng(0)
    dists = []
    for i in range(20):
        Xi = X[off[i]:off[i + 1]]
        a = rng.integers(0, Xi.shape[0], 200)
        b = rng.integers(0, Xi.shape[0], 200)
        dists.append(np.linalg.norm(Xi[a] - Xi[b], axis=1))
    th0 = (float(np.median(np.concatenate(dists))), 0.16, float(np.var(y)))
    return synth.Dataset(X=np.ascontiguousarray(X), y=np.ascontiguousarray(y), offsets=np.asarray(off, dtype=np.int64),
                         reps=np.ascontiguousarray(reps), theta0=th0,
                         meta=dict(config="C4", probe_seed=204, m=8, kernel="matern52", kind="g_real"))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def init_dist(backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend=backend)
    return rank, world, local


# --------------------------------------------------------------------------- oracle timing
def oracle_sample(ds, probe_seed, evals_sel):
    """Time the oracle (as it stands) on the chosen evaluations of one epoch."""
    from oracle.mll import central_perturbations, mll as omll
    from oracle.structured import build_blocks as obuild
    Z = synth.probes(probe_seed, 8, ds.n)
    pts, _ = central_perturbations(ds.theta0, (1e-3,) * 3)
    t0 = time.perf_counter()
    bo = obuild(ds.X, ds.offsets, ds.reps, ds.theta0, ds.meta.get("kernel", "rbf"))
    t_build = time.perf_counter() - t0
    times = {}
    for k in evals_sel:
        t0 = time.perf_counter()
        omll(bo, ds.y, pts[k], Z)
        times[k] = time.perf_counter() - t0
    return t_build, times


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_baseline(ds, probe_seed):
    """Oracle epoch rate estimated from a bounded sample: the build plus one evaluation of each
    operator mode (baseline, noise, scale, generic), extrapolated to the 7 evaluations."""
    t_build, t = oracle_sample(ds, probe_seed, [0, 3, 5, 1])
    epoch = t_build + t[0] + 2 * t[3] + 2 * t[5] + 2 * t[1]
    return {"value": 7.0 / epoch, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": (f"1 build + 4 of the 7 evaluations (one per mode: baseline, noise, scale, "
                       f"lengthscale) at {ds.meta.get('config')}, extrapolated to one epoch of 7; "
                       f"measured {t_build + sum(t.values()):.1f} s, est. epoch {epoch:.1f} s"),
            "host_cores": os.cpu_count()}


def run_reference(args):
    rank, world, _ = init_dist("gloo")
    if rank != 0:
        return
    ds = load_config(args.config)
    seed = ds.meta["probe_seed"]
    from oracle.mll import central_perturbations, mll as omll
    from oracle.structured import build_blocks as obuild
    Z = synth.probes(seed, 8, ds.n)
    pts, _ = central_perturbations(ds.theta0, (1e-3,) * 3)
    state = {"bo": None}

    def step(k):
        if k % 7 == 0 or state["bo"] is None:
            state["bo"] = obuild(ds.X, ds.offsets, ds.reps, ds.theta0, ds.meta.get("kernel", "rbf"))
        omll(state["bo"], ds.y, pts[k % 7], Z)

    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    dt = time.perf_counter() - t0
    value = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}; reference step = one of "
                               "the 7 central-difference MLL evaluations in turn (+ build every 7th)",
                   "parallelism": "cpu-oracle"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
                         "sample": f"{args.steps} timed evaluations after {args.warmup} warm-up"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    rank, world, local = init_dist("nccl")
    torch.cuda.set_device(local)
    import paper_2510_12128_b200 as P
    P._native.lib()
    shard = args.shard == "clusters"
    if shard and world == 1:
        # PAR-2 on one GPU: a 1-rank NCCL group so the exchange path (NCCL all_reduce) is the same
        import socket
        import torch.distributed as dist
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    group = True if (world > 1 or shard) else None
    ctx = P.Context(local, group=group, shard_clusters=shard)
    if args.direct:
        # direct kernel launches instead of the per-evaluation CUDA graphs (for launch tracers / ncu,
        # which cannot see kernels inside conditional graph nodes); same kernels, same results
        ctx.set_option("graphs", False)
    if shard:
        args.eval_slots = 1          # sharded evaluations run one after another, all ranks together
    ds = load_config(args.config, P, ctx)
    kernel = ds.meta.get("kernel", "rbf")
    seed = ds.meta["probe_seed"]
    dev = torch.device("cuda", local)
    Xd = torch.tensor(ds.X, device=dev)
    yd = torch.tensor(ds.y, device=dev)
    rd = torch.tensor(ds.reps, device=dev)
    ws = torch.empty(P.workspace_size(ds.offsets, ds.n_c, ds.d, args.eval_slots, rank, world, shard=shard),
                     dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(local)
    state = np.zeros(10)
    state[:3] = ds.theta0

    def step(st, X, y, reps, epochs=1):
        # `epochs` Algorithm-1 epochs in ONE nugpr_train call (the user-facing training entry)
        st2, rec = P.train(ctx, X, ds.offsets, reps, y, None, epochs=epochs, adam_state=st, workspace=ws,
                           probe_seed=seed, num_probes=8, kernel=kernel, block_storage=args.blocks,
                           logdet=args.logdet)
        return st2, rec

    def barrier():
        if world > 1 or shard:
            import torch.distributed as dist
            dist.barrier()

    # warm-up
    st = state.copy()
    st, _ = step(st, Xd, yd, rd, epochs=args.warmup)
    torch.cuda.synchronize()
    barrier()
    # timed region (device-resident inputs): production mode (CUDA graphs, concurrent slots)
    clocks = ClockSampler(local)
    clocks.start()
    n0 = P.launch_count()
    st = state.copy()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    ev0.record(stream)
    st, recs = step(st, Xd, yd, rd, epochs=args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = P.launch_count() - n0
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 7.0 * args.steps / (ms * 1e-3)
    # e2e: the same public call with HOST buffers (inputs staged H2D inside, records read back)
    Xh, yh, rh = ds.X, ds.y, ds.reps
    st = state.copy()
    step(st, Xh, yh, rh)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):         # one call per step: every step uploads its X, y, reps
        st, _ = step(st, Xh, yh, rh)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    # phase split of one epoch in production mode: the build alone, then the numerical gradient
    phase = {}
    try:
        th0 = tuple(float(t) for t in ds.theta0)
        reps_ph = 3
        e0p, e1p = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0p.record(stream)
        for _ in range(reps_ph):
            blk = P.build_blocks(ctx, Xd, ds.offsets, rd, th0, kernel=kernel, workspace=ws, eval_slots=args.eval_slots)
        e1p.record(stream)
        torch.cuda.synchronize()
        phase["build_ms"] = e0p.elapsed_time(e1p) / reps_ph
        e0p.record(stream)
        for _ in range(reps_ph):
            P.numgrad(ctx, blk, yd, th0, probe_seed=seed, num_probes=8, block_storage=args.blocks,
                      logdet=args.logdet)
        e1p.record(stream)
        torch.cuda.synchronize()
        phase["numgrad_ms"] = e0p.elapsed_time(e1p) / reps_ph
        # each of the 7 central-difference evaluations ALONE on the GPU (its latency: what one rank
        # of the perturbation-sharded gradient waits for; input of DESIGN §7's scaling model)
        if not shard and world == 1:
            l_, s_, a_ = th0
            pts = [th0]
            for i_ in range(3):
                for sg in (1, -1):
                    p_ = [l_, s_, a_]
                    p_[i_] = p_[i_] + sg * 1e-3 * p_[i_]
                    pts.append(tuple(p_))
            solo = []
            for th in pts:
                P.mll(ctx, blk, yd, th, probe_seed=seed, num_probes=8, block_storage=args.blocks, logdet=args.logdet)
                e0p.record(stream)
                for _ in range(reps_ph):
                    P.mll(ctx, blk, yd, th, probe_seed=seed, num_probes=8, block_storage=args.blocks,
                          logdet=args.logdet)
                e1p.record(stream)
                torch.cuda.synchronize()
                solo.append(round(e0p.elapsed_time(e1p) / reps_ph, 4))
            phase["solo_eval_ms"] = solo        # [theta, l+, l-, noise+, noise-, scale+, scale-]
        blk.close()
    except Exception as ex:  # noqa: BLE001
        phase["error"] = str(ex)[:200]
    # Algorithm 1 end to end at the paper's 50 epochs (the "train time" of the metric):
    # ONE nugpr_train call, device-resident inputs, CUDA events around it
    train50 = None
    if args.train_epochs > 0:
        st = state.copy()
        e0t, e1t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier()
        e0t.record(stream)
        step(st, Xd, yd, rd, epochs=args.train_epochs)
        e1t.record(stream)
        torch.cuda.synchronize()
        train50 = e0t.elapsed_time(e1t) / 1e3
    # roofline pass: the same steps with per-kernel CUDA events (direct, serialised launches on
    # the context stream — events cannot bracket kernels inside a graph), after the timed region
    ctx.set_profiling(True)
    st = state.copy()
    st, _ = step(st, Xd, yd, rd, epochs=args.prof_steps)
    torch.cuda.synchronize()
    prof = ctx.profile()
    ctx.set_profiling(False)
    h2d = ds.X.nbytes + ds.y.nbytes + ds.reps.nbytes
    d2h = 7 * 128 + 4 * ds.n_c + 16 + 8 * 10
    # roofline of the dominant kernel: the fused apply with a block term
    peak, peak_src = peaks()
    a_ms, a_bytes, a_n = prof["apply_B"]
    achieved = (a_bytes / (a_ms * 1e-3)) / 1e9 if a_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and args.blocks == "f64" and not shard:
        try:
            traffic = json.load(open(tp)).get(args.config, {}).get("apply_B_dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    total_prof_ms = sum(v[0] for v in prof.values())
    shares = {k: round(v[0] / total_prof_ms, 4) for k, v in prof.items() if total_prof_ms > 0}
    if rank != 0:
        return
    kys = [int(r[7]) for r in recs]
    kqs = [int(r[8]) for r in recs]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.blocks == "f64" else "f64 (FP32-stored H/G blocks)", "data": "synthetic",
        "config": {
            "workload": f"{args.config}: {CONFIG_DESC[args.config]}; step = one Algorithm-1 epoch "
                        "(build preconditioner + 7-point central-difference gradient + Adam)",
            "n": ds.n, "n_c": ds.n_c, "b": int(ds.offsets[1]), "b_max": int(np.diff(ds.offsets).max()), "d": ds.d, "m": 8,
            "kernel": kernel, "logdet": args.logdet, "block_storage": args.blocks,
            "parallelism": (f"cluster-sharded x{world} (PAR-2: contiguous cluster ranges, 3 allreduces of "
                            "per-cluster partials per CG iteration)") if shard else
                           (f"perturbation-sharded x{world}" if world > 1 else "single GPU"),
            "l2": "inputs larger than L2: per step the factor Linv (full) and the packed H, G(lambda+), "
                  "G(lambda-) blocks stream "
                  f"{8 * float(np.sum(np.diff(ds.offsets).astype(np.float64) ** 2)) / 1e6 + 3 * 4 * float(np.sum(np.diff(ds.offsets).astype(np.float64) ** 2)) / 1e6:.0f} MB (> 126 MB L2)",
            "train_time_s": train50, "train_epochs": args.train_epochs,
            "peak_hbm_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
            "dense_n2_f64_gb": 8.0 * ds.n * ds.n / 1e9,
            "cg_iters_y_max": max(kys), "cg_iters_q_max": max(kqs),
            "eval_slots": args.eval_slots,
            "phase_ms": phase,
        },
        "clocks": clk,
        "gpu_launches": int(launches),
        "roofline": {
            "kernel": "apply_packed_kernel (fused multi-RHS matvec of the packed symmetric blocks on the FP64 DMMA "
                      "pipe + in-kernel low-rank correction, modes with a block term)",
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "launches": int(a_n), "avg_launch_us": 1e3 * a_ms / a_n if a_n else None,
            "bytes_per_launch": a_bytes / a_n if a_n else None, "peak_source": peak_src,
            "step_share": shares,
            "how": f"CUDA events around every launch on the context stream in a separate profiling pass of "
                   f"{args.prof_steps} steps (direct serialised launches; the timed region runs CUDA graphs "
                   "with concurrent evaluation streams, where per-kernel events are not available)",
        },
        "e2e": {"value": 7.0 * args.steps / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ds, seed)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--eval-slots", type=int, default=7)
    ap.add_argument("--prof-steps", type=int, default=2)
    ap.add_argument("--blocks", default="f64", choices=["f64", "f32"],
                    help="storage of the streamed blocks H/G (f32: reading X6 fast path, 1e-3 bar)")
    ap.add_argument("--logdet", default="pade", choices=["pade", "slq", "mbcg"],
                    help="log-det estimator (mbcg: NEXT-4, one CG on A, SLQ with f = log)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--direct", action="store_true",
                    help="direct kernel launches instead of the per-evaluation CUDA graphs (ncu launch lists)")
    ap.add_argument("--train-epochs", type=int, default=50,
                    help="also time one nugpr_train call of this many epochs (PAPER.md:404: 50); 0 = skip")
    ap.add_argument("--shard", default="perturbation", choices=["perturbation", "clusters"],
                    help="multi-GPU split: PAR-1 by perturbation (default) or PAR-2 by cluster range")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        pass


if __name__ == "__main__":
    main()
