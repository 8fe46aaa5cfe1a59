"""Build libmpsm_b200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1207_0145_b200.build [--force] [--verbose]

Each csrc/*.cu / *.cpp is compiled to an object under build/ and linked into
paper_1207_0145_b200/libmpsm_b200.so (git-ignored; it travels to the GPU box
with the gpurun snapshot).  nvcc cross-compiles here without a GPU.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "csrc")
LIB = os.path.join(PKG, "libmpsm_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                  "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "mpsm_b200.h"))
    return max(os.path.getmtime(h) for h in hs)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, defines=(), build_dir: str = None,
          lib: str = None) -> str:
    """Compile csrc/ into lib (default: the in-tree libmpsm_b200.so)."""
    BUILD = build_dir or globals()["BUILD"]
    LIB = lib or globals()["LIB"]
    os.makedirs(BUILD, exist_ok=True)
    hdr = _headers_mtime()
    objs, jobs = [], []
    for src in _sources():
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(sp), hdr):
            extra = ["-Xptxas", "-v"] if ptxas_info and src.endswith(".cu") else []
            cmd = [NVCC] + CUFLAGS + [f"-D{d}" for d in defines] + extra + ["-c", sp, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-x", "c++", "-c", sp, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                print(err)
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        run(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
