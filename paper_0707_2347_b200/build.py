"""Build the native library ``libwinomem_b200.so`` in-tree for sm_100a (and
``libwinomem_b200_diag.so``: the same library plus the measurement-only probes
and wm_diag_* exports that scripts/ and one kernel-level test use).

    python -m paper_0707_2347_b200.build        (or __graft_entry__.build())

nvcc cross-compiles every CUDA / C++ source under csrc/ with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and links one shared
library next to this file (it travels to the GPU box with the repo snapshot).
Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libwinomem_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", CSRC, "-I", INC,
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
# measurement builds only (e.g. WM_NVCC_FLAGS=-DWM_EPI_MODE=1); never set for the product
COMMON += os.environ.get("WM_NVCC_FLAGS", "").split()


# measurement-only probes: linked into libwinomem_b200_diag.so, never the product
DIAG_ONLY = {"wm_diag.cu"}
DIAG_LIB = os.path.join(HERE, "libwinomem_b200_diag.so")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(CSRC, "*.inc")) + glob.glob(os.path.join(INC, "*.h")))


def _compile(job, hdr_mtime, verbose):
    src, diag = job
    obj = os.path.join(OBJ, os.path.basename(src) + (".diag.o" if diag else ".o"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    flags = COMMON + (["-DWM_DIAG=1"] if diag else [])
    cmd = [NVCC] + ARCH + flags + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-x", "cu"] + ARCH + flags + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose=False, jobs=None):
    os.makedirs(OBJ, exist_ok=True)
    from . import gen_fusion  # schedule-specific fused addition kernels
    gen_fusion.main()
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    srcs = _sources()
    runtime = os.path.join(CSRC, "wm_runtime.cu")
    jobs_ = [(s_, False) for s_ in srcs] + [(runtime, True)]
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 1)) as ex:
        objs = dict(zip(jobs_, ex.map(lambda j: _compile(j, hdr_mtime, verbose), jobs_)))
    product = [objs[(s_, False)] for s_ in srcs if os.path.basename(s_) not in DIAG_ONLY]
    diag = [objs[(s_, False)] for s_ in srcs if s_ != runtime] + [objs[(runtime, True)]]
    for lib, parts in ((LIB, product), (DIAG_LIB, diag)):
        if os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(o) for o in parts):
            continue
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + parts
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_0707_2347_b200 import build as _b
    print(_b.build(verbose="-v" in sys.argv))
