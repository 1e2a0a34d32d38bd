"""In-tree build of `_hdgb.so` for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2007_11891_b200.build [--force]

Each translation unit in csrc/ is compiled in parallel to build/*.o, then
linked into paper_2007_11891_b200/_hdgb.so with a static CUDA runtime.
"""

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# HDGB_BUILD_TAG / HDGB_DEFS: side builds for tuning experiments (build_<tag>/, _hdgb_<tag>.so,
# extra -D definitions); the product build uses neither
_TAG = os.environ.get("HDGB_BUILD_TAG", "")
BUILD = os.path.join(ROOT, "build" + (f"_{_TAG}" if _TAG else ""))
OUT = os.path.join(HERE, f"_hdgb_{_TAG}.so" if _TAG else "_hdgb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "hdgb.h")]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in _deps())


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *os.environ.get("HDGB_DEFS", "").split(), "-c", src, "-o", obj]
    if os.environ.get("HDGB_PTXAS_VERBOSE"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    # the library is stamped with the newest source time seen at the START of the build, so a
    # source edited while nvcc runs still counts as newer than the library
    t_src = max(os.path.getmtime(p) for p in _deps())
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(_compile, _sources()))
    if verbose:
        for _, log in results:
            if log.strip():
                print(log)
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp] + [o for o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    os.utime(OUT, (t_src, t_src))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
