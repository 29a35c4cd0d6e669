"""Build the sm_100a CUDA library in-tree (no JIT cache, no torch extension).

    python -m paper_1908_10396_b200.build      # -> paper_1908_10396_b200/libanisoq_b200.so

Every .cu under csrc/ is compiled with
`nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo` and linked into
one shared library whose exported symbols are exactly the C ABI declared in
include/anisoq_b200.h. The CUDA runtime is linked statically so the .so only
needs the driver on the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "libanisoq_b200.so")
CLI = os.path.join(PKG, "anisoq_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
         "-I", os.path.join(ROOT, "include")] + os.environ.get("AQ_NVCC_FLAGS", "").split()


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_digest() -> str:
    h = hashlib.sha1()
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cuh", ".h")):
            h.update(open(os.path.join(CSRC, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "anisoq_b200.h"), "rb").read())
    return h.hexdigest()


def _compile(src: str, hdr: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    stamp = obj + ".stamp"
    key = hashlib.sha1(open(path, "rb").read() + hdr.encode() +
                       " ".join(ARCH + FLAGS).encode()).hexdigest()
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == key:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    open(stamp, "w").write(key)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr = _headers_digest()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), _sources()))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cli()
    return LIB


def build_cli() -> str:
    """The anisoq_b200 command-line tool (cli/anisoq_b200_main.cpp) over the C++
    drop-in headers, linked against the in-tree library (rpath $ORIGIN)."""
    src = os.path.join(PKG, "cli", "anisoq_b200_main.cpp")
    deps = [src, LIB] + [os.path.join(ROOT, "include", "anisoq", f)
                         for f in os.listdir(os.path.join(ROOT, "include", "anisoq"))]
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(f) for f in deps):
        return CLI
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), src,
           "-o", CLI, "-L", PKG, "-lanisoq_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
