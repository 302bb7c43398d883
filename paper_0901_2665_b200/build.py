"""In-tree build of libfeastgpu.so (sm_100a only) — called by __graft_entry__.build().

Each translation unit is compiled to its own object in parallel (paper_0901_2665_b200/build/,
git-ignored) and only the ones whose source or headers changed are rebuilt; the objects are then
linked into the shared library with the CUDA runtime linked statically."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libfeastgpu.so")
SOURCES = ["blocktri.cu", "sweep.cu", "sweep_small.cu", "sweep_pipe.cu", "sweep_tma.cu", "gemm.cu", "band_apply.cu",
           "dense.cu", "chol.cu", "chol_tiles.cu", "eig.cu", "tridiag.cu", "tridiag_tiles.cu",
           "tri_back.cu", "misc.cu", "csr_ingest.cu", "bicgstab.cu", "spike.cu", "feast_gpu.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC"]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static", "-Xlinker", "-soname=libfeastgpu.so"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(os.path.dirname(HERE), "include", "feast_gpu.h"))
    return hs


def _obj(src):
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _stale(src, newest_header):
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return os.path.getmtime(os.path.join(CSRC, src)) > t or newest_header > t


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + _headers()
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    newest = max(os.path.getmtime(h) for h in _headers())
    todo = [s for s in SOURCES if force or _stale(s, newest)]

    def compile_one(src):
        cmd = [nvcc(), *COMPILE_FLAGS, "-c", "-o", _obj(src), os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}{r.stderr}")
        return src

    with cf.ThreadPoolExecutor(max_workers=jobs or min(len(todo) or 1, os.cpu_count() or 4)) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    cmd = [nvcc(), *LINK_FLAGS, "-o", LIB, *[_obj(s) for s in SOURCES], "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose=True)
