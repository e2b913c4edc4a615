"""paper_2510_12128_b200 — B200-native nuGPR MLL hot path (arXiv 2510.12128).

Thin Python binding over the C-ABI of libnugpr.so (include/nugpr.h): argument marshalling
only.  Every step of the MLL evaluation runs in the library's sm_100a CUDA kernels; PyTorch
provides device memory (the workspace tensor), the stream and the process group.

    ctx = Context(device=0)
    cl = cluster(ctx, X, n_c, y=y)                                               # row A0
    blocks = build_blocks(ctx, X_sorted, offsets, reps, theta0, kernel="rbf")   # row A1
    rec = mll(ctx, blocks, y_sorted, theta)                                      # rows A2-A7
    L0, g, evals = numgrad(ctx, blocks, y_sorted, theta)                         # row A8
    state, records = train(ctx, X_sorted, offsets, reps, y_sorted, theta0)      # row A9
"""
from __future__ import annotations

import ctypes as C
import os

# More hardware work queues than the default 8 for the concurrent evaluation streams (effective
# when this package is imported before CUDA is initialised in the process).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np

from . import _native as N
from ._native import NugprError

__all__ = ["Context", "Blocks", "cluster", "build_blocks", "predict", "mll", "numgrad", "train", "adam_step",
           "shard_plan", "tridiag_eig", "workspace_size", "NugprError", "version"]


def version() -> str:
    return N.lib().nugpr_version().decode()


def launch_count() -> int:
    """Kernel launches issued by libnugpr.so in this process."""
    return int(N.lib().nugpr_launch_count())


def _ptr(x, keep):
    """Pointer to a float64/int64 C-contiguous torch tensor (any device) or numpy array."""
    if x is None:
        return None
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                raise ValueError("tensor must be contiguous")
            keep.append(x)
            return x.data_ptr()
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(x)
    keep.append(a)
    return a.ctypes.data


def _f64(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.float64:
                raise TypeError("expected float64 tensor")
            return x.contiguous()
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(x, dtype=np.float64)


def _theta(t):
    return N.Theta(float(t[0]), float(t[1]), float(t[2]))


class Context:
    """nugpr_ctx on one device, enqueuing on torch's current stream of that device.

    group: an initialised torch.distributed process group (or True for the default group)
    enables perturbation sharding in numgrad/train via the allgather callback (PAR-1).
    shard_clusters=True additionally (PAR-2) keeps only this rank's cluster range in the blocks
    and makes mll/numgrad/train collective over the group.

    comm: "nccl" — the library creates its own NCCL communicator (nugpr_ctx_set_nccl; torch only
    broadcasts the 128-byte id) and runs every exchange as an NCCL collective on the context
    stream, captured into the evaluation graphs; "callback" — the exchanges go through
    torch.distributed from Python callbacks (gloo groups: CPU tests, several ranks on one GPU).
    Default: "nccl" when the group's backend is NCCL, else "callback"."""

    def __init__(self, device: int = 0, stream=None, group=None, shard_clusters: bool = False, comm=None):
        """device < 0: host-only context (rank/world/allgather for the host helpers; no CUDA)."""
        self.device = int(device)
        self.rank, self.world = 0, 1
        self.group = None
        if group is not None:
            import torch.distributed as dist
            self.group = None if group is True else group
            self.rank = dist.get_rank(self.group)
            self.world = dist.get_world_size(self.group)
        if self.device >= 0:
            import torch
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            sp = C.c_void_p(stream.cuda_stream)
        else:
            sp = C.c_void_p(None)
        self.stream = stream
        h = C.c_void_p()
        N.check(N.lib().nugpr_ctx_create(self.device, sp, self.rank, self.world, C.byref(h)))
        self.handle = h
        self._cb = None
        self.comm = None
        if group is not None and self.device >= 0:
            import torch.distributed as dist
            if comm is None:
                comm = "nccl" if dist.get_backend(self.group) == "nccl" else "callback"
            self.comm = comm
            if comm == "nccl":
                import torch
                # the library's own communicator: rank 0 creates the id, torch broadcasts its bytes
                idb = (C.c_uint8 * N.NCCL_ID_BYTES)()
                if self.rank == 0:
                    N.check(N.lib().nugpr_nccl_unique_id(idb))
                t = torch.tensor(list(bytes(idb)), dtype=torch.uint8, device=torch.device("cuda", self.device))
                dist.broadcast(t, src=dist.get_global_rank(self.group, 0) if self.group is not None else 0,
                               group=self.group)
                idb = (C.c_uint8 * N.NCCL_ID_BYTES)(*t.cpu().tolist())
                N.check(N.lib().nugpr_ctx_set_nccl(self.handle, idb))
            elif comm != "callback":
                raise ValueError(f"comm must be 'nccl' or 'callback', not {comm!r}")
        if self.world > 1 and self.comm != "nccl":
            self._cb = N.ALLGATHER_FN(self._allgather)
            N.check(N.lib().nugpr_ctx_set_allgather(self.handle, self._cb, None))
        self.shard_clusters = bool(shard_clusters)
        self._buffers = {}          # data_ptr -> tensor: device memory the exchange may address
        self._ar_cb = None
        self.exchanges = 0
        if self.shard_clusters:
            if group is None:
                raise ValueError("shard_clusters needs a torch.distributed process group")
            if self.comm == "nccl":
                N.check(N.lib().nugpr_ctx_set_option(self.handle, N.OPTIONS["shard_clusters"], 1))
            else:
                self._ar_cb = N.ALLREDUCE_FN(self._allreduce)
                N.check(N.lib().nugpr_ctx_set_cluster_shard(self.handle, self._ar_cb, None))

    def sharded_graphs(self) -> bool:
        """True if sharded evaluations run their CG loop as one captured graph with the library's
        NCCL exchanges inside (nugpr_ctx_sharded_graphs)."""
        return bool(N.lib().nugpr_ctx_sharded_graphs(self.handle))

    def register(self, buf):
        """Make a tensor's memory addressable by the PAR-2 exchange (build_blocks does this for
        its workspace)."""
        self._buffers[buf.data_ptr()] = buf

    def _view(self, ptr, count):
        import torch
        nb = 8 * count
        for base, buf in self._buffers.items():
            size = buf.numel() * buf.element_size()
            if base <= ptr and ptr + nb <= base + size:
                off = ptr - base
                return buf.view(torch.uint8)[off:off + nb].view(torch.float64)
        # host memory (host-only tests): wrap without copying
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(count,))
        return torch.from_numpy(arr)

    def _allreduce(self, send, recv, count, stream, user):
        """PAR-2 exchange: recv = sum over ranks of send, ordered on the context stream."""
        try:
            import contextlib
            import torch
            import torch.distributed as dist
            s_t, r_t = self._view(send, count), self._view(recv, count)
            # order the copies / collective on the stream the library enqueued its partials on (the
            # caller's current torch stream may be another one)
            sc = (torch.cuda.stream(torch.cuda.ExternalStream(stream, device=torch.device("cuda", self.device)))
                  if (r_t.is_cuda and stream) else contextlib.nullcontext())
            with sc:
                if r_t.is_cuda and dist.get_backend(self.group) != "nccl":
                    # gloo (CPU tests, or several ranks sharing one GPU): through host memory
                    tmp = s_t.cpu()
                    dist.all_reduce(tmp, group=self.group)
                    r_t.copy_(tmp)
                else:
                    r_t.copy_(s_t)
                    dist.all_reduce(r_t, group=self.group)
            self.exchanges += 1
            return 0
        except Exception as exc:  # noqa: BLE001 — reported to C as a status
            import sys
            print(f"[nugpr] PAR-2 allreduce failed: {exc!r}", file=sys.stderr)
            return 1

    def _allgather(self, send, nbytes, recv, user):
        try:
            data = allgather_bytes(C.string_at(send, nbytes), self.world, self.group, self.device)
            C.memmove(recv, data, len(data))
            return 0
        except Exception:  # noqa: BLE001 — reported to C as a status
            return 1

    def set_option(self, name: str, value):
        """nugpr_ctx_set_option: 'graphs' (CG loop as a device-driven CUDA graph, default True)."""
        N.check(N.lib().nugpr_ctx_set_option(self.handle, N.OPTIONS[name], int(value)))

    def set_profiling(self, enable: bool = True):
        N.check(N.lib().nugpr_ctx_set_profiling(self.handle, int(bool(enable))))

    def profile(self) -> dict:
        """{class: (ms, algorithmic_bytes, launches)} accumulated since set_profiling(True)."""
        out = {}
        for name, cls in N.PROF_CLASSES.items():
            ms, by, n = C.c_double(), C.c_double(), C.c_int64()
            N.check(N.lib().nugpr_ctx_profile(self.handle, cls, C.byref(ms), C.byref(by), C.byref(n)))
            out[name] = (ms.value, by.value, n.value)
        return out

    def close(self):
        if getattr(self, "handle", None):
            N.lib().nugpr_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


def cluster(ctx: Context, X, n_c: int, y=None, init_centers=None, seed: int = 0, max_iter: int = 100,
            rep_mode: str = "centroid", kernel: str = "rbf", theta=(1.0, 0.1, 1.0)) -> dict:
    """Row A0: k-means + stable cluster sort.  Returns device tensors
    perm, reps, X_sorted, y_sorted (if y given), host offsets and the iteration count."""
    import torch
    keep = []
    Xf = _f64(X)
    n, d = int(Xf.shape[0]), int(Xf.shape[1])
    dev = torch.device("cuda", ctx.device)
    nb = C.c_size_t()
    N.check(N.lib().nugpr_cluster_workspace_size(n, d, int(n_c), C.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    reps = torch.empty((n_c, d), dtype=torch.float64, device=dev)
    Xs = torch.empty((n, d), dtype=torch.float64, device=dev)
    ys = torch.empty(n, dtype=torch.float64, device=dev) if y is not None else None
    off = np.zeros(n_c + 1, dtype=np.int64)
    it = C.c_int32(0)
    N.check(N.lib().nugpr_cluster(ctx.handle, _ptr(Xf, keep), n, d, int(n_c),
                                  _ptr(_f64(init_centers), keep) if init_centers is not None else None,
                                  int(seed) & 0xFFFFFFFFFFFFFFFF, int(max_iter), N.REP_MODES[rep_mode],
                                  N.KERNELS[kernel], _theta(theta),
                                  _ptr(_f64(y), keep) if y is not None else None,
                                  C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(perm.data_ptr()),
                                  off.ctypes.data, C.c_void_p(reps.data_ptr()), C.c_void_p(Xs.data_ptr()),
                                  C.c_void_p(ys.data_ptr()) if ys is not None else None, C.byref(it)))
    return dict(perm=perm, offsets=off, reps=reps, X_sorted=Xs, y_sorted=ys, iters=int(it.value))


def allgather_bytes(data: bytes, world: int, group=None, device: int = -1) -> bytes:
    """Allgather of equal-length byte strings through torch.distributed (NCCL on GPU boxes with
    a CUDA device, gloo on CPU): the rank-ordered concatenation."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device) if (backend == "nccl" and device >= 0) else torch.device("cpu")
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
    out = torch.empty(world * len(data), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.cpu().numpy().tobytes()


def numgrad_exchange(ctx: Context, theta, step, L_mine, status_mine=None):
    """Host side of the perturbation-sharded CENTRAL gradient (nugpr_numgrad_exchange).  Raises
    NugprError with the exchanged worst status when any evaluation (of any rank) failed."""
    st = np.ascontiguousarray(step, dtype=np.float64)
    Lm = np.ascontiguousarray(L_mine, dtype=np.float64)
    sm = None if status_mine is None else np.ascontiguousarray(status_mine, dtype=np.int32)
    L0 = C.c_double()
    g = np.zeros(3)
    P_ = C.POINTER(C.c_double)
    N.check(N.lib().nugpr_numgrad_exchange(ctx.handle, _theta(theta), st.ctypes.data_as(P_), Lm.ctypes.data_as(P_),
                                           sm.ctypes.data if sm is not None else None, C.byref(L0),
                                           g.ctypes.data_as(P_)))
    return L0.value, g


def workspace_size(offsets, n_c: int, d: int, eval_slots: int = 1, rank: int = 0, world: int = 1,
                   shard: bool = False) -> int:
    """Workspace bytes (shard=True: this rank's PAR-2 cluster range, nugpr_workspace_size_shard)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    out = C.c_size_t()
    if shard:
        N.check(N.lib().nugpr_workspace_size_shard(off.ctypes.data, int(n_c), int(d), int(eval_slots), int(rank),
                                                   int(world), C.byref(out)))
    else:
        N.check(N.lib().nugpr_workspace_size(off.ctypes.data, int(n_c), int(d), int(eval_slots), C.byref(out)))
    return int(out.value)


def shard_range(offsets, rank: int, world: int):
    """PAR-2: the cluster range [lo, hi) rank `rank` of `world` holds (balanced by sum ld_i^2)."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    r = (C.c_int32 * 2)()
    N.check(N.lib().nugpr_shard_range(off.ctypes.data, off.shape[0] - 1, int(rank), int(world), r))
    return int(r[0]), int(r[1])


def _ctx_workspace(ctx, off, n_c, d, eval_slots):
    import torch
    nbytes = workspace_size(off, n_c, d, eval_slots, ctx.rank, ctx.world, getattr(ctx, "shard_clusters", False))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", ctx.device))
    return ws


class Blocks:
    """nugpr_blocks handle + the torch workspace it lives in."""

    def __init__(self, ctx, handle, ws, offsets, d, theta0, kernel, jitter, failed):
        self.ctx, self.handle, self.workspace = ctx, handle, ws
        self.offsets = offsets
        self.n = int(offsets[-1])
        self.n_c = int(offsets.shape[0] - 1)
        self.d = d
        self.theta0 = tuple(float(t) for t in theta0)
        self.kernel = kernel
        self.max_jitter = jitter

    def export(self, what: str):
        """Debug read-back (tests): 'linv', 'H', 'u', 'jitter', 'scalars', 'M', 'ld', 'probes'."""
        codes = {"linv": 0, "H": 1, "u": 2, "jitter": 3, "scalars": 4, "M": 5, "ld": 6, "probes": 7}
        ld = np.zeros(self.n_c, dtype=np.int32)
        N.check(N.lib().nugpr_blocks_export(self.handle, 6, ld.ctypes.data, ld.nbytes))
        if what == "ld":
            return ld
        if what in ("linv", "H"):
            tot = int(np.sum(ld.astype(np.int64) ** 2))
            buf = np.empty(tot)
            N.check(N.lib().nugpr_blocks_export(self.handle, codes[what], buf.ctypes.data, buf.nbytes))
            out, pos = [], 0
            for i in range(self.n_c):
                l = int(ld[i])
                b = int(self.offsets[i + 1] - self.offsets[i])
                blk = buf[pos:pos + l * l].reshape(l, l).T          # col-major -> [row, col]
                out.append(blk[:b, :b].copy())
                pos += l * l
            return out
        sizes = {"u": self.n, "jitter": self.n_c, "scalars": 2, "M": self.n_c * self.n_c}
        if what == "probes":
            raise ValueError("use export_probes(m)")
        buf = np.empty(sizes[what])
        N.check(N.lib().nugpr_blocks_export(self.handle, codes[what], buf.ctypes.data, buf.nbytes))
        return buf.reshape(self.n_c, self.n_c) if what == "M" else buf

    def lanczos_info(self, which: str = "build"):
        """(iterations, converged) of the build's lambda_0 solve or of the last generic eval's."""
        buf = np.zeros(2, dtype=np.int32)
        N.check(N.lib().nugpr_blocks_export(self.handle, 8 if which == "build" else 9, buf.ctypes.data,
                                            buf.nbytes))
        return int(buf[0]), bool(buf[1])

    def export_probes(self, m: int):
        buf = np.empty((m, self.n))
        N.check(N.lib().nugpr_blocks_export(self.handle, 7, buf.ctypes.data, buf.nbytes))
        return buf

    def close(self):
        if getattr(self, "handle", None):
            N.lib().nugpr_blocks_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


def build_blocks(ctx: Context, X_sorted, offsets, reps, theta0, kernel: str = "rbf",
                 eval_slots: int = 1, workspace=None) -> Blocks:
    """Row A1 (Alg. 1): preconditioner, u_i, H_i, K_rep, lambda_0 at theta0."""
    import torch
    keep = []
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    X = _f64(X_sorted)
    n_c, d = off.shape[0] - 1, int(X.shape[1])
    if workspace is None:
        workspace = _ctx_workspace(ctx, off, n_c, d, eval_slots)
    if getattr(ctx, "shard_clusters", False):
        ctx.register(workspace)
    h = C.c_void_p()
    fb = C.c_int32(-1)
    jit = C.c_double(0.0)
    st = N.lib().nugpr_build_blocks(ctx.handle, _ptr(X, keep), off.ctypes.data, n_c, d,
                                    _ptr(_f64(reps), keep), N.KERNELS[kernel], _theta(theta0),
                                    C.c_void_p(workspace.data_ptr()), workspace.numel(), C.byref(h),
                                    C.byref(fb), C.byref(jit))
    N.check(st)
    return Blocks(ctx, h, workspace, off, d, theta0, kernel, jit.value, fb.value)


def _solve_cfg(num_probes=8, tol=0.01, max_iter=2000, probe_seed=0, probes=None, replay=None,
               logdet="pade", block_storage="f64", keep=None):
    cfg = N.SolveCfg()
    cfg.cg_tol = float(tol)
    cfg.cg_max_iter = int(max_iter)
    cfg.num_probes = int(num_probes)
    cfg.probe_seed = int(probe_seed) & 0xFFFFFFFFFFFFFFFF
    cfg.probes = _ptr(_f64(probes), keep) if probes is not None else None
    if replay is not None:
        r = np.ascontiguousarray(replay, dtype=np.int32)
        keep.append(r)
        cfg.replay_iters = r.ctypes.data
    cfg.logdet_mode = {"pade": 0, "slq": 1, "mbcg": 2}[logdet]
    cfg.block_storage = {"f64": 0, "f32": 1}[block_storage]
    return cfg


def _rec(o: N.MllOut, m: int) -> dict:
    return dict(L=o.L, quad=o.quad, logdet=o.logdet, logdet_pade=o.logdet_pade,
                logdet_slq=o.logdet_slq, logdet_R=o.logdet_R, lambda0=o.lambda0,
                resid_y=o.resid_y, resid_q_max=o.resid_q_max, iters_y=o.iters_y,
                iters_q=[o.iters_q[j] for j in range(m)], iters_q_max=o.iters_q_max,
                converged=bool(o.converged), mode=N.MODES.get(o.mode, o.mode), breakdown=bool(o.breakdown),
                lanczos_iters=o.lanczos_iters, lanczos_converged=bool(o.lanczos_converged),
                lambda0_degenerate=bool(o.lambda0_degenerate),
                probe_t=[o.probe_t[j] for j in range(m)], probe_s=[o.probe_s[j] for j in range(m)])


def mll(ctx: Context, blocks: Blocks, y_sorted, theta, **solve) -> dict:
    """Rows A2-A7: one MLL evaluation (Alg. 1 ComputeLoss) at theta."""
    keep = []
    cfg = _solve_cfg(keep=keep, **solve)
    out = N.MllOut()
    N.check(N.lib().nugpr_mll(ctx.handle, blocks.handle, _ptr(_f64(y_sorted), keep), _theta(theta),
                              C.byref(cfg), C.byref(out)))
    return _rec(out, cfg.num_probes)


def predict(ctx: Context, blocks: Blocks, y_sorted, X_test, add_noise: bool = False, variance: bool = True):
    """NEXT-1: posterior mean (and variance) at the blocks' theta0 (Eq. 4-5, exact structured
    K''^{-1}).  Returns device tensors (mean, var or None)."""
    import torch
    keep = []
    Xt = _f64(X_test)
    n_t = int(Xt.shape[0])
    dev = torch.device("cuda", ctx.device)
    mean = torch.empty(n_t, dtype=torch.float64, device=dev)
    var = torch.empty(n_t, dtype=torch.float64, device=dev) if variance else None
    N.check(N.lib().nugpr_predict(ctx.handle, blocks.handle, _ptr(_f64(y_sorted), keep), _ptr(Xt, keep), n_t,
                                  int(bool(add_noise)), C.c_void_p(mean.data_ptr()),
                                  C.c_void_p(var.data_ptr()) if var is not None else None))
    return mean, var


def mll_exact(ctx: Context, blocks: Blocks, y_sorted) -> dict:
    """NEXT-2: the exact structured MLL at the blocks' theta0 (determinant lemma + Woodbury on
    Eq. (28)-(29); no probes, Pade or CG)."""
    keep = []
    out = (C.c_double * 4)()
    N.check(N.lib().nugpr_mll_exact(ctx.handle, blocks.handle, _ptr(_f64(y_sorted), keep), out))
    return {"L": out[0], "quad": out[1], "logdet": out[2], "logdet_C": out[3]}


def _grad_cfg(mode="central", step=None, threshold=1e-3, threshold_relative=True, max_halvings=20):
    g = N.GradCfg()
    g.mode = {"central": 0, "forward_halving": 1}[mode]
    if step is None:
        step = (1e-3, 1e-3, 1e-3) if mode == "central" else (0.1, 0.1, 0.1)
    for i in range(3):
        g.step[i] = float(step[i])
    g.threshold = float(threshold)
    g.threshold_relative = int(bool(threshold_relative))
    g.max_halvings = int(max_halvings)
    return g


def numgrad(ctx: Context, blocks: Blocks, y_sorted, theta, mode="central", step=None,
            threshold=1e-3, threshold_relative=True, max_halvings=20, **solve):
    """Row A8: numerical gradient (CENTRAL 2p+1 = 7 evaluations, or FORWARD_HALVING)."""
    keep = []
    scfg = _solve_cfg(keep=keep, **solve)
    gcfg = _grad_cfg(mode, step, threshold, threshold_relative, max_halvings)
    L0 = C.c_double()
    g = (C.c_double * 3)()
    cap = 1 + 3 * 21
    evals = (N.MllOut * cap)()
    ne = C.c_int32(0)
    N.check(N.lib().nugpr_numgrad(ctx.handle, blocks.handle, _ptr(_f64(y_sorted), keep), _theta(theta),
                                  C.byref(gcfg), C.byref(scfg), C.byref(L0), g, evals, C.byref(ne)))
    return L0.value, np.array(list(g)), [_rec(evals[k], scfg.num_probes) for k in range(ne.value)]


def train(ctx: Context, X_sorted, offsets, reps, y_sorted, theta0, epochs=50, lr=0.05,
          kernel="rbf", adam_state=None, mode="central", step=None, threshold=1e-3,
          threshold_relative=True, max_halvings=20, eval_slots=1, workspace=None, **solve):
    """Row A9: Algorithm 1 (build blocks, numerical gradient, Adam) for `epochs` epochs."""
    import torch
    keep = []
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    X = _f64(X_sorted)
    n_c, d = off.shape[0] - 1, int(X.shape[1])
    if workspace is None:
        workspace = _ctx_workspace(ctx, off, n_c, d, eval_slots)
    if getattr(ctx, "shard_clusters", False):
        ctx.register(workspace)
    scfg = _solve_cfg(keep=keep, **solve)
    gcfg = _grad_cfg(mode, step, threshold, threshold_relative, max_halvings)
    st = np.zeros(10)
    if adam_state is None:
        st[:3] = theta0
    else:
        st[:] = adam_state
    rec = np.zeros((max(epochs, 1), N.NUGPR_TRAIN_RECORD))
    N.check(N.lib().nugpr_train(ctx.handle, _ptr(X, keep), off.ctypes.data, n_c, d, _ptr(_f64(reps), keep),
                                _ptr(_f64(y_sorted), keep), N.KERNELS[kernel], int(epochs), float(lr),
                                C.byref(gcfg), C.byref(scfg), st.ctypes.data_as(C.POINTER(C.c_double)),
                                C.c_void_p(rec.ctypes.data), C.c_void_p(workspace.data_ptr()),
                                workspace.numel()))
    return st, rec[:epochs]


def adam_step(state, grad, lr=0.05):
    s = np.ascontiguousarray(state, dtype=np.float64).copy()
    g = np.ascontiguousarray(grad, dtype=np.float64)
    N.check(N.lib().nugpr_adam_step(s.ctypes.data_as(C.POINTER(C.c_double)),
                                    g.ctypes.data_as(C.POINTER(C.c_double)), float(lr)))
    return s


def shard_plan(world: int, costs):
    c = np.ascontiguousarray(costs, dtype=np.float64)
    owner = np.zeros(c.shape[0], dtype=np.int32)
    N.check(N.lib().nugpr_shard_plan(int(world), c.ctypes.data_as(C.POINTER(C.c_double)), c.shape[0],
                                     owner.ctypes.data_as(C.POINTER(C.c_int32))))
    return owner


def tridiag_eig(diag, off):
    d = np.ascontiguousarray(diag, dtype=np.float64)
    e = np.ascontiguousarray(off, dtype=np.float64) if len(off) else np.zeros(1)
    k = d.shape[0]
    ev, first = np.zeros(k), np.zeros(k)
    P = C.POINTER(C.c_double)
    N.check(N.lib().nugpr_tridiag_eig(k, d.ctypes.data_as(P), e.ctypes.data_as(P), ev.ctypes.data_as(P),
                                      first.ctypes.data_as(P)))
    return ev, first
