"""Multi-process (world_size 2 and 3, gloo on CPU) tests of the perturbation-sharded numerical
gradient's host side (PAR-1): every rank computes the same LPT shard plan, owns
a subset of the 7 CENTRAL evaluations, exchanges its records with ONE allgather through the
library's callback (routed through torch.distributed), and all ranks must return the identical
L0 and gradient.  The evaluations are replaced by a closed-form loss so the test needs no GPU;
nugpr_numgrad runs the same exchange (central_exchange) after its device evaluations."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

THETA = (0.7, 0.16, 1.3)
STEP = (1e-3, 2e-3, 5e-4)
COSTS = [1.0, 3.0, 3.0, 2.0, 2.0, 2.0, 2.0]


def loss(t):
    l, s, a = t
    return 3.0 * l * l - 2.0 * l * s + 5.0 * s * s + a * a * a + 7.0


def points():
    th = np.array(THETA)
    h = np.array(STEP) * th
    pts = [tuple(th)]
    for i in range(3):
        for sg in (1.0, -1.0):
            p = th.copy()
            p[i] = th[i] + sg * h[i]
            pts.append(tuple(p))
    return pts, h


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_12128_b200 as P
        ctx = P.Context(-1, group=True)
        owner = P.shard_plan(world, COSTS)
        pts, _ = points()
        L_mine = [loss(pts[k]) if owner[k] == rank else float("nan") for k in range(7)]
        L0, g = P.numgrad_exchange(ctx, THETA, STEP, L_mine)
        q.put((rank, L0, g.tolist(), owner.tolist(), None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_central_gradient_exchange_gloo(world):
    from paper_2510_12128_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        from paper_2510_12128_b200 import build
        build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for r in res:
        assert r[4] is None, r[4]
    pts, h = points()
    want_g = [(loss(pts[1 + 2 * i]) - loss(pts[2 + 2 * i])) / (2.0 * h[i]) for i in range(3)]
    owners = res[0][3]
    assert sorted(set(owners)) == list(range(world))            # every rank owns something
    for rank, L0, g, own, _ in res:
        assert own == owners                                    # same plan on every rank
        assert L0 == loss(THETA)                                # bit-exact exchange
        assert g == want_g                                      # identical on every rank
    # the central difference of this polynomial is its gradient up to O(h^2) (cubic in alpha)
    l, s, a = THETA
    exact = [6 * l - 2 * s, -2 * l + 10 * s, 3 * a * a]
    np.testing.assert_allclose(res[0][2], exact, rtol=1e-5)


def test_single_rank_exchange_needs_no_collective():
    import paper_2510_12128_b200 as P
    ctx = P.Context(-1)
    pts, h = points()
    L0, g = P.numgrad_exchange(ctx, THETA, STEP, [loss(p) for p in pts])
    assert L0 == loss(THETA)
    assert list(g) == [(loss(pts[1 + 2 * i]) - loss(pts[2 + 2 * i])) / (2.0 * h[i]) for i in range(3)]


def _worker_fail(rank, world, port, q):
    """Rank 1 reports a hard failure (NOT_SPD = 3) for the first evaluation it owns and
    CG_NOT_CONVERGED (5) for another; every rank must return the same worst status together."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_12128_b200 as P
        ctx = P.Context(-1, group=True)
        owner = P.shard_plan(world, COSTS)
        pts, _ = points()
        L_mine = [loss(pts[k]) if owner[k] == rank else float("nan") for k in range(7)]
        st = [0] * 7
        mine = [k for k in range(7) if owner[k] == rank]
        if rank == 1:
            st[mine[-1]] = 5
            st[mine[0]] = 3
        try:
            P.numgrad_exchange(ctx, THETA, STEP, L_mine, status_mine=st)
            q.put((rank, None, "no error raised"))
        except P.NugprError as e:
            q.put((rank, e.name, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_failed_evaluation_fails_every_rank_together():
    """a rank whose evaluation fails must not return before the PAR-1 exchange (the
    others would wait forever in the allgather).  The statuses travel with the records, so every
    rank returns the same error, the hard failure (NOT_SPD) winning over CG_NOT_CONVERGED."""
    from paper_2510_12128_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        from paper_2510_12128_b200 import build
        build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fail, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[2] for r in res] == [None, None], res
    assert [r[1] for r in res] == ["NOT_SPD", "NOT_SPD"]
