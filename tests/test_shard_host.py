"""PAR-2 host side, no GPU: the cluster partition (nugpr_shard_range), the per-rank
workspace (nugpr_workspace_size_shard) and the binding's allreduce callback over gloo at world
size 2 (the same marshalling the device exchange uses, here on host buffers)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def P():
    from paper_2510_12128_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        from paper_2510_12128_b200 import build
        build.build()
    import paper_2510_12128_b200 as pkg
    return pkg


def offsets_of(sizes):
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions_and_balances(P, world):
    rng = np.random.default_rng(world)
    sizes = rng.integers(20, 500, size=57)
    off = offsets_of(sizes)
    cost = ((sizes + 7) // 8 * 8).astype(float) ** 2
    ranges = [P.shard_range(off, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == len(sizes)
    for r in range(world - 1):
        assert ranges[r][1] == ranges[r + 1][0]
    assert all(hi > lo for lo, hi in ranges)
    loads = [cost[lo:hi].sum() for lo, hi in ranges]
    # contiguous split at the nearest prefix boundary: off the ideal share by < one cluster per side
    assert max(loads) <= cost.sum() / world + 2 * cost.max()


def test_shard_range_uniform_clusters_split_evenly(P):
    off = offsets_of([500] * 2000)          # C5
    ranges = [P.shard_range(off, r, 8) for r in range(8)]
    assert [hi - lo for lo, hi in ranges] == [250] * 8


def test_shard_range_rejects_more_ranks_than_clusters(P):
    from paper_2510_12128_b200 import _native as N
    with pytest.raises(N.NugprError):
        P.shard_range(offsets_of([100] * 3), 0, 4)


def test_shard_workspace_sizes(P):
    off = offsets_of([500] * 64)
    full = P.workspace_size(off, 64, 4, 1)
    assert P.workspace_size(off, 64, 4, 1, 0, 1, shard=True) >= full   # + exchange buffers
    per = [P.workspace_size(off, 64, 4, 1, r, 8, shard=True) for r in range(8)]
    # blocks and vectors split 8 ways; the replicated K_rep / M / exchange arrays are small here
    assert max(per) < full / 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_12128_b200 as P
        ctx = P.Context(-1, group=True, shard_clusters=True)
        n = 37
        send = np.zeros(n)
        lo, hi = (0, 20) if rank == 0 else (20, n)
        send[lo:hi] = np.arange(lo, hi) * 0.5 + rank      # own slots only, zeros elsewhere
        recv = np.full(n, np.nan)
        st = ctx._allreduce(send.ctypes.data, recv.ctypes.data, n, None, None)
        q.put((rank, st, recv.tolist(), None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_allreduce_callback_gloo_world2(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    expect = np.arange(37) * 0.5 + (np.arange(37) >= 20)
    for rank, st, recv, err in res:
        assert err is None, err
        assert st == 0
        assert np.array_equal(np.array(recv), expect)     # exact: x + 0 = x
