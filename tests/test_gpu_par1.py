"""PAR-1: perturbation-sharded central-difference gradient with REAL device
evaluations.  Each rank evaluates the 2p+1 = 7 points its LPT share (nugpr_shard_plan) assigns to
it on its own blocks and the records are allgathered; every rank then forms the same L0, gradient
and Adam step.

Only one GPU is available, so the world-size 2 and 3 runs put every rank on cuda:0 with the gloo
backend (the allgather goes through the binding's callback); the world-size 1 NCCL run uses the
library's own communicator (nugpr_ctx_set_nccl).  An evaluation does not depend on which rank runs
it or on what else runs concurrently (fixed reduction orders), so the sharded gradient must equal
the replicated one-GPU gradient BIT FOR BIT, and so must two epochs of Algorithm 1."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    ds = synth.g_hyper(n_c=24, b=200, d=8, seed=117)
    return ds.X, ds.y, ds.offsets, ds.reps, tuple(ds.theta0)


def _run(P, ctx):
    X, y, off, reps, th0 = _case()
    bg = P.build_blocks(ctx, X, off, reps, th0, eval_slots=7)
    L0, g, ev = P.numgrad(ctx, bg, y, th0, probe_seed=9)
    bg.close()
    st, rec = P.train(ctx, X, off, reps, y, th0, epochs=2, probe_seed=9)
    return dict(L0=L0, g=[float(v) for v in g], L=[e["L"] for e in ev], iters=[e["iters_y"] for e in ev],
                state=[float(v) for v in st], rec=np.asarray(rec).tolist())


def _worker(rank, world, port, backend, q, comm):
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
        ctx = P.Context(0, group=True, comm=comm)
        q.put((rank, _run(P, ctx), None))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _spawn(world, backend, comm):
    import torch.multiprocessing as mp
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    procs = [mctx.Process(target=_worker, args=(r, world, port, backend, q, comm)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    res.sort(key=lambda t: t[0])
    for r, out, err in res:
        assert err is None, f"rank {r}:\n{err}"
    return [out for _, out, _ in res]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_12128_b200 as pkg
    pkg._native.lib()
    return pkg


@pytest.fixture(scope="module")
def replicated(P):
    return _run(P, P.Context(0))


@pytest.mark.parametrize("world,backend,comm", [(2, "gloo", "callback"), (3, "gloo", "callback"),
                                                (1, "nccl", "nccl")])
def test_par1_gradient_and_training_equal_replicated_bitwise(P, replicated, world, backend, comm):
    outs = _spawn(world, backend, comm)
    for out in outs:
        assert out["L0"] == replicated["L0"]
        assert out["g"] == replicated["g"]
        assert out["L"] == replicated["L"] and out["iters"] == replicated["iters"]
        assert out["state"] == replicated["state"]
        assert out["rec"] == replicated["rec"]
