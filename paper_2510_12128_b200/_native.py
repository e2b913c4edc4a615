"""ctypes declarations of include/nugpr.h (argument marshalling only).

The CUDA library is mandatory: if libnugpr.so is missing or fails to load, every entry point
raises — there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnugpr.so")

NUGPR_MAX_PROBES = 15
NUGPR_NUM_EVALS = 7
NUGPR_TRAIN_RECORD = 12

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "SHAPE", 3: "NOT_SPD", 4: "DEGENERATE_REPS",
          5: "CG_NOT_CONVERGED", 6: "WORKSPACE", 7: "CUDA", 8: "COMM", 9: "INTERNAL",
          10: "UNSUPPORTED", 11: "BREAKDOWN"}
KERNELS = {"rbf": 0, "matern52": 1, "rbf_as_printed": 2}
REP_MODES = {"given": 0, "centroid": 1, "medoid": 2}
MODES = {0: "baseline", 1: "noise", 2: "scale", 3: "generic"}
OPTIONS = {"graphs": 0, "shard_clusters": 1}
NCCL_ID_BYTES = 128
PROF_CLASSES = {"apply_B": 0, "apply_lowrank": 1, "update": 2, "rhs": 3, "gemm": 4, "chol": 5,
                "lanczos": 6, "other": 7}


class NugprError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"nugpr {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Theta(C.Structure):
    _fields_ = [("lengthscale", C.c_double), ("noise", C.c_double), ("outputscale", C.c_double)]


class SolveCfg(C.Structure):
    _fields_ = [("cg_tol", C.c_double), ("cg_max_iter", C.c_int32), ("num_probes", C.c_int32),
                ("probe_seed", C.c_uint64), ("probes", C.c_void_p), ("replay_iters", C.c_void_p),
                ("logdet_mode", C.c_int32), ("block_storage", C.c_int32)]


class GradCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("max_halvings", C.c_int32), ("step", C.c_double * 3),
                ("threshold", C.c_double), ("threshold_relative", C.c_int32), ("reserved", C.c_int32)]


class MllOut(C.Structure):
    _fields_ = [("L", C.c_double), ("quad", C.c_double), ("logdet", C.c_double),
                ("logdet_pade", C.c_double), ("logdet_slq", C.c_double), ("logdet_R", C.c_double),
                ("lambda0", C.c_double), ("resid_y", C.c_double), ("resid_q_max", C.c_double),
                ("iters_y", C.c_int32), ("iters_q_max", C.c_int32), ("iters_q", C.c_int32 * 16),
                ("converged", C.c_int32), ("mode", C.c_int32), ("breakdown", C.c_int32),
                ("lanczos_iters", C.c_int32), ("lanczos_converged", C.c_int32), ("lambda0_degenerate", C.c_int32),
                ("probe_t", C.c_double * 16), ("probe_s", C.c_double * 16)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
# nugpr_allreduce_fn(send, recv, count, stream, user) — PAR-2 cluster sharding
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)

_lib = None


def lib():
    """Load libnugpr.so (raises if absent: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2510_12128_b200.build` "
                          "(or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "nugpr_version": (C.c_char_p, []),
        "nugpr_last_error": (C.c_char_p, []),
        "nugpr_ctx_create": (C.c_int, [C.c_int, P, C.c_int, C.c_int, C.POINTER(P)]),
        "nugpr_ctx_set_allgather": (C.c_int, [P, ALLGATHER_FN, P]),
        "nugpr_ctx_set_cluster_shard": (C.c_int, [P, ALLREDUCE_FN, P]),
        "nugpr_shard_range": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
        "nugpr_workspace_size_shard": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_size_t)]),
        "nugpr_ctx_destroy": (C.c_int, [P]),
        "nugpr_ctx_set_profiling": (C.c_int, [P, C.c_int32]),
        "nugpr_ctx_set_option": (C.c_int, [P, C.c_int32, C.c_int32]),
        "nugpr_ctx_profile": (C.c_int, [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int64)]),
        "nugpr_launch_count": (C.c_int64, []),
        "nugpr_workspace_size": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
        "nugpr_build_blocks": (C.c_int, [P, P, P, C.c_int32, C.c_int32, P, C.c_int32, Theta, P,
                                         C.c_size_t, C.POINTER(P), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_double)]),
        "nugpr_blocks_destroy": (C.c_int, [P]),
        "nugpr_blocks_export": (C.c_int, [P, C.c_int32, P, C.c_size_t]),
        "nugpr_mll": (C.c_int, [P, P, P, Theta, C.POINTER(SolveCfg), C.POINTER(MllOut)]),
        "nugpr_numgrad": (C.c_int, [P, P, P, Theta, C.POINTER(GradCfg), C.POINTER(SolveCfg),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(MllOut),
                                    C.POINTER(C.c_int32)]),
        "nugpr_train": (C.c_int, [P, P, P, C.c_int32, C.c_int32, P, P, C.c_int32, C.c_int32,
                                  C.c_double, C.POINTER(GradCfg), C.POINTER(SolveCfg),
                                  C.POINTER(C.c_double), P, P, C.c_size_t]),
        "nugpr_cluster_workspace_size": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
        "nugpr_cluster": (C.c_int, [P, P, C.c_int64, C.c_int32, C.c_int32, P, C.c_uint64, C.c_int32,
                                    C.c_int32, C.c_int32, Theta, P, P, C.c_size_t, P, P, P, P, P,
                                    C.POINTER(C.c_int32)]),
        "nugpr_numgrad_exchange": (C.c_int, [P, Theta, C.POINTER(C.c_double), C.POINTER(C.c_double), P,
                                             C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "nugpr_predict": (C.c_int, [P, P, P, P, C.c_int64, C.c_int32, P, P]),
        "nugpr_mll_exact": (C.c_int, [P, P, P, C.POINTER(C.c_double)]),
        "nugpr_adam_step": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double]),
        "nugpr_shard_plan": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int32)]),
        "nugpr_tridiag_eig": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "nugpr_nccl_unique_id": (C.c_int, [P]),
        "nugpr_ctx_set_nccl": (C.c_int, [P, P]),
        "nugpr_ctx_sharded_graphs": (C.c_int32, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int):
    if status != 0:
        raise NugprError(status, lib().nugpr_last_error().decode())


EXPORTED = ["nugpr_version", "nugpr_last_error", "nugpr_ctx_create", "nugpr_ctx_set_allgather",
            "nugpr_ctx_destroy", "nugpr_ctx_set_profiling", "nugpr_ctx_profile",
            "nugpr_launch_count", "nugpr_workspace_size", "nugpr_build_blocks", "nugpr_blocks_destroy",
            "nugpr_blocks_export", "nugpr_mll", "nugpr_numgrad", "nugpr_train", "nugpr_adam_step",
            "nugpr_shard_plan", "nugpr_tridiag_eig", "nugpr_cluster_workspace_size", "nugpr_cluster",
            "nugpr_numgrad_exchange", "nugpr_predict", "nugpr_mll_exact", "nugpr_ctx_set_cluster_shard",
            "nugpr_shard_range", "nugpr_workspace_size_shard", "nugpr_ctx_set_option",
            "nugpr_nccl_unique_id", "nugpr_ctx_set_nccl", "nugpr_ctx_sharded_graphs"]
