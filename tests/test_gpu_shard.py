"""PAR-2: cluster-sharded evaluation.  Each rank holds a contiguous cluster range
(its blocks, vectors and partials) and the CG runs collectively with three exchanges of
zero-padded per-cluster partial arrays per iteration (S(A p) of the low-rank term, p^T q, and
r^T r with S(r)), routed through torch.distributed.all_reduce.

Only one GPU is available to this build, so the world-size 2 / 3 runs put every rank on cuda:0
with the gloo backend (the binding moves the partials through host memory); the world-size 1
run uses the NCCL backend, exercising the device-side all_reduce path of the same callback.
The exchange is exact (every rank's partials land in their own slots, zeros elsewhere), so a
sharded evaluation must reproduce the replicated single-GPU evaluation — which is itself
parity-tested against the oracle — to the last bit or to FP64 reduction-order noise; the
tests assert 1e-12 relative, identical CG iteration counts, identical records on every rank,
and the oracle (replay mode) at the 1e-9 bar on the baseline evaluation."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TIGHT = 1e-12


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dataset(case):
    if case == "C5":
        ds = synth.make_config("C5")
        return ds.X, ds.y, ds.offsets, ds.reps, tuple(ds.theta0)
    if case == "uneven":
        rng = np.random.default_rng(7)
        sizes = rng.integers(60, 400, size=13)
        d = 3
        reps = rng.uniform(-10, 10, size=(len(sizes), d))
        X = np.concatenate([reps[i] + 0.8 * rng.standard_normal((s, d)) for i, s in enumerate(sizes)])
        y = np.sin(X).sum(axis=1) + 0.4 * rng.standard_normal(X.shape[0])
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        return X, y, off, reps, (1.1, 0.16, 1.0)
    ds = synth.g_hyper(n_c=40, b=200, d=8, seed=113)
    return ds.X, ds.y, ds.offsets, ds.reps, tuple(ds.theta0)


def variants(P, ctx):
    """Jitter ladder, NOT_SPD agreement, FP32 block storage and FORWARD_HALVING under the same
    context (sharded or not)."""
    from paper_2510_12128_b200 import _native as N
    out = {}
    rng = np.random.default_rng(2)
    X = np.concatenate([rng.normal(size=(12, 2)), 5 + rng.normal(size=(12, 2)), np.zeros((12, 2)),
                        -5 + rng.normal(size=(12, 2))])
    y = rng.normal(size=48)
    off = np.array([0, 12, 24, 36, 48], dtype=np.int64)
    reps = np.array([[0.0, 0.0], [5.0, 5.0], [0.0, 0.0], [-5.0, -5.0]]) + np.array([[0, 0], [0, 0], [0.0, 9.0], [0, 0]])
    th0 = (1.0, 1e-18, 1.0)
    bg = P.build_blocks(ctx, X, off, reps, th0)          # cluster 2 (identical points) needs jitter
    out["max_jitter"] = bg.max_jitter
    out["jitter_mll"] = P.mll(ctx, bg, y, th0, probe_seed=9, tol=1e-6)
    bg.close()
    Xn = X.copy()
    Xn[40] = np.nan                                        # cluster 3 cannot be factorised
    try:
        P.build_blocks(ctx, Xn, off, reps, (1.0, 0.1, 1.0))
        out["not_spd"] = None
    except N.NugprError as e:
        out["not_spd"] = e.name
    Xc, yc, offc, repsc, thc = dataset("c3shape")
    bg = P.build_blocks(ctx, Xc, offc, repsc, thc)
    out["f32"] = P.mll(ctx, bg, yc, (thc[0], thc[1] * 1.001, thc[2]), probe_seed=5, block_storage="f32")
    L0, g, ev = P.numgrad(ctx, bg, yc, thc, probe_seed=5, mode="forward_halving")
    out["halving"] = dict(L0=L0, g=g.tolist(), n=len(ev))
    bg.close()
    return out


def run_all(P, ctx, case):
    if case == "variants":
        return variants(P, ctx)
    X, y, off, reps, th0 = dataset(case)
    bg = P.build_blocks(ctx, X, off, reps, th0)
    out = {}
    if case == "C5":                  # full size: one evaluation per operator mode family
        out["pade"] = P.mll(ctx, bg, y, th0, probe_seed=205)
        out["noise"] = P.mll(ctx, bg, y, (th0[0], th0[1] * 1.001, th0[2]), probe_seed=205)
        out["lam"] = P.mll(ctx, bg, y, (th0[0] * 1.001, th0[1], th0[2]), probe_seed=205)
        out["scalars"] = [float(v) for v in bg.export("scalars")]
        bg.close()
        return out
    out["pade"] = P.mll(ctx, bg, y, th0, probe_seed=5)
    out["slq"] = P.mll(ctx, bg, y, th0, probe_seed=5, logdet="slq")
    L0, g, ev = P.numgrad(ctx, bg, y, th0, probe_seed=5)
    out["numgrad"] = dict(L0=L0, g=g.tolist(), evals=ev)
    out["scalars"] = [float(v) for v in bg.export("scalars")]
    bg.close()
    st, rec = P.train(ctx, X, off, reps, y, th0, epochs=2, probe_seed=5)
    out["train"] = dict(state=st.tolist(), rec=rec.tolist())
    return out


def _worker(rank, world, port, backend, case, q, comm=None):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_12128_b200 as P
        ctx = P.Context(0, group=True, shard_clusters=True, comm=comm)
        out = run_all(P, ctx, case)
        out["sharded_graphs"] = ctx.sharded_graphs()
        if case != "variants":
            out["range"] = P.shard_range(dataset(case)[2], rank, world)
        out["exchanges"] = ctx.exchanges
        q.put((rank, out, None))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_12128_b200 as pkg
    pkg._native.lib()
    return pkg


def spawn(world, backend, case, comm=None):
    import torch.multiprocessing as mp
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    procs = [mctx.Process(target=_worker, args=(r, world, port, backend, case, q, comm)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    res.sort(key=lambda t: t[0])
    for r, out, err in res:
        assert err is None, f"rank {r}:\n{err}"
    return [out for _, out, _ in res]


def same_rec(a, b, tol=TIGHT):
    assert a["iters_y"] == b["iters_y"] and a["iters_q"] == b["iters_q"], (a, b)
    assert a["mode"] == b["mode"]
    for k in ("L", "quad", "logdet_pade", "logdet_slq", "logdet_R", "lambda0"):
        assert rel(a[k], b[k]) <= tol, (k, a[k], b[k])


def check_against_replicated(P, outs, case):
    ctx = P.Context(0)
    ref = run_all(P, ctx, case)
    for out in outs:
        same_rec(out["pade"], ref["pade"])
        same_rec(out["slq"], ref["slq"])
        assert rel(out["numgrad"]["L0"], ref["numgrad"]["L0"]) <= TIGHT
        np.testing.assert_allclose(out["numgrad"]["g"], ref["numgrad"]["g"], rtol=1e-9, atol=1e-12)
        for a, b in zip(out["numgrad"]["evals"], ref["numgrad"]["evals"]):
            same_rec(a, b)
        np.testing.assert_allclose(out["scalars"], ref["scalars"], rtol=TIGHT)
        np.testing.assert_allclose(out["train"]["state"], ref["train"]["state"], rtol=1e-9)
    # every rank returns the identical records (the CG state is replicated)
    for out in outs[1:]:
        assert out["pade"]["L"] == outs[0]["pade"]["L"]
        assert out["numgrad"]["g"] == outs[0]["numgrad"]["g"]
    return ref


def check_oracle(outs, case):
    from oracle import structured as OS
    from oracle.mll import mll as oracle_mll
    X, y, off, reps, th0 = dataset(case)
    bo = OS.build_blocks(X, off, reps, th0)
    rec = outs[0]["pade"]
    Z = synth.probes(5, 8, y.shape[0])
    ro = oracle_mll(bo, y, th0, Z, replay=[rec["iters_y"]] + list(rec["iters_q"]))
    for k in ("L", "quad", "logdet_pade", "logdet_slq"):
        assert rel(rec[k], getattr(ro, k)) < 1e-9, (k, rec[k], getattr(ro, k))


@pytest.mark.parametrize("world,case", [(2, "uneven"), (3, "c3shape")])
def test_cluster_shard_gloo_matches_replicated(P, world, case):
    outs = spawn(world, "gloo", case)
    ranges = [o["range"] for o in outs]
    assert ranges[0][0] == 0 and all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
    assert all(o["exchanges"] > 0 for o in outs)
    check_against_replicated(P, outs, case)
    check_oracle(outs, case)


def test_cluster_shard_nccl_world1(P):
    """Real NCCL group at world 1: the library's own communicator (nugpr_ctx_set_nccl; no Python
    exchange callback runs, the sharded CG loop is one captured graph with the NCCL collectives
    inside) and the callback route through torch.distributed both equal the replicated path."""
    outs = spawn(1, "nccl", "c3shape", comm="nccl")
    assert outs[0]["exchanges"] == 0
    assert outs[0]["sharded_graphs"], "the NCCL exchanges were not captured into the evaluation graph"
    check_against_replicated(P, outs, "c3shape")
    outs = spawn(1, "nccl", "c3shape", comm="callback")
    assert outs[0]["exchanges"] > 0 and not outs[0]["sharded_graphs"]
    check_against_replicated(P, outs, "c3shape")


def test_cluster_shard_C5_full_size_world4(P):
    """C5 (n = 1M, 2000 clusters x 500) split over 4 ranks (500 clusters each; gloo, all on cuda:0):
    baseline, noise-step and lengthscale-step evaluations equal the replicated one-GPU path."""
    outs = spawn(4, "gloo", "C5")
    assert [o["range"] for o in outs] == [(0, 500), (500, 1000), (1000, 1500), (1500, 2000)]
    ctx = P.Context(0)
    X, y, off, reps, th0 = dataset("C5")
    bg = P.build_blocks(ctx, X, off, reps, th0)
    ref = {"pade": P.mll(ctx, bg, y, th0, probe_seed=205),
           "noise": P.mll(ctx, bg, y, (th0[0], th0[1] * 1.001, th0[2]), probe_seed=205),
           "lam": P.mll(ctx, bg, y, (th0[0] * 1.001, th0[1], th0[2]), probe_seed=205)}
    scal = [float(v) for v in bg.export("scalars")]
    bg.close()
    for out in outs:
        for k in ("pade", "noise", "lam"):
            same_rec(out[k], ref[k])
        np.testing.assert_allclose(out["scalars"], scal, rtol=TIGHT)


def test_cluster_shard_variants_world2(P):
    """Under PAR-2 (world 2): the jitter ladder's outcome is shared (rank 1 owns the singular
    cluster, both report the same largest jitter), a block that cannot be factorised fails on
    EVERY rank with NOT_SPD (no rank is left waiting in an exchange), FP32 block storage and the
    FORWARD_HALVING gradient equal the replicated path."""
    outs = spawn(2, "gloo", "variants")
    ref = variants(P, P.Context(0))
    assert ref["max_jitter"] > 0 and ref["not_spd"] == "NOT_SPD"
    for out in outs:
        assert out["max_jitter"] == ref["max_jitter"]
        assert out["not_spd"] == "NOT_SPD"
        same_rec(out["jitter_mll"], ref["jitter_mll"], tol=1e-10)
        same_rec(out["f32"], ref["f32"])
        assert out["halving"]["n"] == ref["halving"]["n"]
        assert rel(out["halving"]["L0"], ref["halving"]["L0"]) <= TIGHT
        np.testing.assert_allclose(out["halving"]["g"], ref["halving"]["g"], rtol=1e-9, atol=1e-12)
