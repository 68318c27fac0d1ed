"""Build libparis.so (the C-ABI library) and the harness datagen library in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a (B200 only; no other targets).
Each .cu is compiled to an object in parallel, then linked with -shared.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libparis.so")
DATAGEN_SRC = os.path.join(ROOT, "datagen", "datagen.cu")
DATAGEN_LIB = os.path.join(ROOT, "datagen", "libparis_datagen.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]
if os.environ.get("PARIS_LB1_SPT"):  # tuning experiments only
    FLAGS = FLAGS + [f"-DPARIS_LB1_SPT={int(os.environ['PARIS_LB1_SPT'])}"]
if os.environ.get("PARIS_LB_NOMAX"):  # tuning experiments only (bit-identical LB accumulation form)
    FLAGS = FLAGS + [f"-DPARIS_LB_NOMAX={int(os.environ['PARIS_LB_NOMAX'])}"]
for _k in ("PARIS_LBI_GROUPS", "PARIS_REF_RUN", "PARIS_REFQ_CTAS", "PARIS_REFU_CTAS", "PARIS_REFU_U", "PARIS_REFU16_CTAS", "PARIS_REFU16_MUL", "PARIS_LBI_UNROLL",
           "PARIS_RAW16_MINLEN", "PARIS_LBI_THREADS", "PARIS_LBI_DYN", "PARIS_BM_CTAS", "PARIS_REFM_CTAS",
           "PARIS_REFM_KP", "PARIS_REFM_H", "PARIS_REFM_ROWS"):  # tuning experiments only
    if os.environ.get(_k):
        FLAGS = FLAGS + [f"-D{_k}={int(os.environ[_k])}"]
if os.environ.get("PARIS_DEBUG"):  # device bounds checks (PARIS_DCHECK) -- debugging builds only
    FLAGS = FLAGS + ["-DPARIS_DEBUG_CHECKS"]
SOURCES = ["runtime.cu", "summarize.cu", "knn.cu", "index.cu", "merge.cu", "select.cu"]
HEADERS = ["runtime.cuh", "gfilter.cuh"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


STAMP = LIB + ".flags"


def _stamp_ok(path: str, flags) -> bool:
    """The library at `path` was built with exactly these flags (tuning -D values included)."""
    try:
        return open(path + ".flags").read() == " ".join(flags)
    except OSError:
        return False


def build_paris(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "paris.h")]
    if not force and not _newer(LIB, deps + [__file__]) and _stamp_ok(LIB, FLAGS):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        extra = ["-Xptxas", "-v"] if verbose else []
        out = _run([NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj])
        return obj, out

    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(compile_one, srcs))
    if verbose:
        for _, out in results:
            sys.stdout.write(out)
    tmp = LIB + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], "-lcudart"])
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:  # a later default build() rebuilds over a tuned (-D...) variant
        f.write(" ".join(FLAGS))
    return LIB


def build_datagen(force: bool = False) -> str:
    if not force and not _newer(DATAGEN_LIB, [DATAGEN_SRC, __file__]) and _stamp_ok(DATAGEN_LIB, FLAGS):
        return DATAGEN_LIB
    tmp = DATAGEN_LIB + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, *FLAGS, "-shared", "-o", tmp, DATAGEN_SRC, "-lcudart"])
    os.replace(tmp, DATAGEN_LIB)
    with open(DATAGEN_LIB + ".flags", "w") as f:
        f.write(" ".join(FLAGS))
    return DATAGEN_LIB


def build_all(force: bool = False, verbose: bool = False):
    return build_paris(force, verbose), build_datagen(force)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
