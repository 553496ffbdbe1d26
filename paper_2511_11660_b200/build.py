"""Build libsta.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsta.so")
SOURCES = ["sta_api.cpp", "sta_kernels.cu", "sta_levelize.cu", "sta_steiner.cu", "sta_arnoldi.cu"]
HEADERS = ["sta_internal.h", "sta_arnoldi.cuh", os.path.join("..", "..", "include", "sta.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-cudart", "static",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, flags: str = "") -> str:
    """Build libsta.so (or, for tuning experiments, a variant at `out` with
    extra nvcc `flags`, e.g. "-DSTA_FWD_THREADS=640")."""
    if out is None and not force and not _stale():
        return LIB
    lib = out or LIB
    odir = os.path.dirname(os.path.abspath(lib))
    os.makedirs(odir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(odir, os.path.basename(lib) + "." + src + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *os.environ.get("STA_NVCC_FLAGS", "").split(), *flags.split(),
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(odir, (os.path.basename(lib) + "." if out else "") + src + ".ptxas.txt"), "w") as f:
            # resources only (compile times would churn the committed report)
            f.write("".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l))
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="variant library path (tuning experiments)")
    ap.add_argument("--flags", default="", help="extra nvcc flags of the variant")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, out=a.out, flags=a.flags))
