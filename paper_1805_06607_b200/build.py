"""Build libmrab.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo
snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libmrab.so")
SOURCES = ["mrab_api.cu", "kernels.cu", "kernels2d.cu", "host_setup.cpp", "dist.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [*(["-DMRAB_Z3_PROF"] if os.environ.get("MRAB_Z3_PROF") else []),
         *([f"-DMRAB_W3_MINB={os.environ['MRAB_W3_MINB']}"] if os.environ.get("MRAB_W3_MINB") else []),
         *([f"-DMRAB_F3_MINB={os.environ['MRAB_F3_MINB']}"] if os.environ.get("MRAB_F3_MINB") else []),
         *([f"-DMRAB_W3_WY={os.environ['MRAB_W3_WY']}"] if os.environ.get("MRAB_W3_WY") else []),
         *([f"-DMRAB_W3_WX={os.environ['MRAB_W3_WX']}"] if os.environ.get("MRAB_W3_WX") else []), "-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    hdr = os.path.join(os.path.dirname(HERE), "include", "mrab.h")
    return os.path.getmtime(hdr) > t


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    # headers are shared by every translation unit: a changed header rebuilds all objects
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "mrab.h"))
    newest_hdr = max(os.path.getmtime(h) for h in hdrs)

    def compile_one(s):
        src = os.path.join(CSRC, s)
        obj = os.path.join(LIBDIR, s + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), newest_hdr)):
            return obj, ""
        cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr}")
        with open(os.path.join(LIBDIR, s + ".ptxas.log"), "w") as f:
            f.write(r.stderr)
        return obj, r.stderr

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in res]
    if verbose:
        for _, e in res:
            sys.stderr.write(e)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB,
           "-Xcompiler", "-fopenmp", "-cudart", "static", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
