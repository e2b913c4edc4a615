"""Build libnugpr.so in-tree for sm_100a with nvcc (no GPU needed; nvcc cross-compiles).

    python -m paper_2510_12128_b200.build [--verbose]

Produces paper_2510_12128_b200/libnugpr.so (git-ignored; it travels to the GPU box with the
gpurun snapshot).  Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnugpr.so")
SOURCES = ["api.cu", "build_kernels.cu", "eval_kernels.cu", "apply_kernels.cu", "cluster_kernels.cu", "big_kernels.cu",
           "predict_kernels.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(INCLUDE, "nugpr.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_v: bool = False, trace: bool = False) -> str:
    """trace=True: the diagnostics variant libnugpr_trace.so (per-CTA globaltimer stamps of one
    packed apply, tools/apply_trace.py); never loaded by the package itself."""
    build_dir = BUILD + ("_trace" if trace else "")
    lib_path = LIB.replace(".so", "_trace.so") if trace else LIB
    extra = ["-DNUGPR_TRACE_APPLY"] if trace else []
    os.makedirs(build_dir, exist_ok=True)
    nv = nvcc()
    hdrs = _headers()
    objs = []
    jobs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if _stale(obj, [sp] + hdrs):
            cmd = [nv, *ARCH, *FLAGS, *extra, "-c", sp, "-o", obj]
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if verbose or res.returncode != 0 or ptxas_v:
                sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    if _stale(lib_path, objs):
        cmd = [nv, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib_path, *objs, "-cudart", "static"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError("link failed")
    return lib_path


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, ptxas_v="--ptxas" in sys.argv, trace="--trace" in sys.argv))
