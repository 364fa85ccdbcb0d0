"""Build libgalois.so in-tree with nvcc for sm_100a (B200) only.

    python -m paper_2603_28796_b200.build [--force] [-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# developer knobs for A/B builds: extra nvcc flags, and a separate object dir / library path
EXTRA = os.environ.get("GALOIS_NVCC_EXTRA", "").split()
OBJ = os.environ.get("GALOIS_OBJ_DIR", os.path.join(ROOT, "build", "obj"))
LIB = os.environ.get("GALOIS_LIB_OUT", os.path.join(PKG, "libgalois.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-ftz=true", "-Xcompiler", "-fPIC,-O2,-Wall", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
SOURCES = ["cnf_build.cu", "step_kernels.cu", "clause_kernels.cu", "update_kernels.cu", "soft_kernels.cu",
           "select_kernels.cu", "tseitin_kernels.cu", "engine.cu", "comm.cpp"]
HEADERS = ["galois_internal.h", "philox.cuh", "device_utils.cuh", "comm.h"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "galois.h"),
                                                               os.path.abspath(__file__)]
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = r.stdout + r.stderr
    with open(obj + ".log", "w") as f:
        f.write(log)
    if verbose:
        print(log)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if any(f.startswith("-DGALOIS_PARITY_BREAKING_EXPERIMENT") for f in EXTRA) and LIB == os.path.join(PKG, "libgalois.so"):
        raise RuntimeError("parity-breaking experiment builds must go to their own GALOIS_LIB_OUT, "
                           "never to the product libgalois.so")
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in SOURCES if force or _stale(os.path.join(OBJ, s + ".o"), os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [os.path.join(OBJ, s + ".o") for s in SOURCES]
    if force or todo or not os.path.exists(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
