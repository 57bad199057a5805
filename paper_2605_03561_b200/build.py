"""Builds libpsg.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

The extension is a plain shared library with a C ABI (include/psg.h); Python
binds it with ctypes (paper_2605_03561_b200/_lib.py).  Objects are cached by
mtime so repeated builds are cheap.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libpsg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", f"-I{ROOT}/include", f"-I{CSRC}"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    headers += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    jobs = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if f.endswith(".cu"):
            cmd = [NVCC, *ARCH, *COMMON, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "--expt-relaxed-constexpr", "-c", src, "-o", obj]
        elif f.endswith(".cpp"):
            cmd = ["g++", *COMMON, "-fPIC", "-Wall", "-Wextra", "-I/usr/local/cuda/include",
                   "-c", src, "-o", obj]
        else:
            continue
        jobs.append((obj, cmd, _stale(obj, [src, *headers])))
    with ThreadPoolExecutor(max_workers=4) as ex:
        for (obj, cmd, stale), out in zip(jobs, ex.map(lambda j: _run(j[1]) if j[2] else "", jobs)):
            if verbose and out:
                sys.stderr.write(out)
    objs = [j[0] for j in jobs]
    if _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl", "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
