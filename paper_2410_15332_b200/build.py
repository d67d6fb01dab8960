"""Build libpic.so in-tree: nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_2410_15332_b200.build [-v]

Objects go to build/ (git-ignored), the shared library to paper_2410_15332_b200/libpic.so
(git-ignored, but it travels to the GPU box with gpurun)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", os.environ.get("PIC_OBJ_DIR", "obj"))
LIB = os.path.join(PKG, os.environ.get("PIC_LIB_NAME", "libpic.so"))  # name override: experiment builds only
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", INCLUDE, "-I", CSRC,
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    out = [os.path.join(CSRC, "engine.cpp"), os.path.join(CSRC, "serve.cpp"), os.path.join(CSRC, "testhooks.cpp")]
    kd = os.path.join(CSRC, "kernels")
    out += sorted(os.path.join(kd, f) for f in os.listdir(kd) if f.endswith(".cu"))
    return out


def headers():
    hs = [os.path.join(INCLUDE, "pic.h"), os.path.join(INCLUDE, "pic_test.h")]
    for d, _, fs in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in fs if f.endswith((".h", ".cuh"))]
    return hs


def _obj(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(OBJ, rel + ".o")


def _compile(src: str, verbose: bool) -> str:
    o = _obj(src)
    cmd = [nvcc(), *ARCH, *FLAGS, *os.environ.get("PIC_NVCC_EXTRA", "").split(), "-c", src, "-o", o]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)
    return o


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    hmax = max(os.path.getmtime(h) for h in headers())
    todo = [s for s in srcs if force or not os.path.exists(_obj(s))
            or os.path.getmtime(_obj(s)) < max(os.path.getmtime(s), hmax, os.path.getmtime(__file__))]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [_obj(s) for s in srcs]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
