"""Build libsq.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2312_03788_b200.build [--force] [--verbose]

Object files are rebuilt when their source or any header is newer.  The result
is paper_2312_03788_b200/_lib/libsq.so (git-ignored, but shipped to the GPU box
with the repo snapshot).
"""

from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libsq.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    f"-I{os.path.join(ROOT, 'include')}",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _newer(src: str, dst: str, deps) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in [src, *deps])


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, defines=(), name: str = "") -> str:
    """Compile every csrc/*.cu and link libsq.so.  `defines`/`name` build a tuning variant
    into _lib/variants/libsq_<name>.so (development only)."""
    obj_dir = OBJ_DIR if not name else os.path.join(OUT_DIR, "obj_" + name)
    lib = LIB if not name else os.path.join(OUT_DIR, "variants", f"libsq_{name}.so")
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "libsq.h")]
    objs = []
    for src in sources:
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _newer(src, obj, headers):
            cmd = [nvcc(), *CFLAGS, *dflags, "-c", src, "-o", obj]
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
            if verbose or ptxas_v:
                sys.stderr.write(r.stderr)
    if force or any(_newer(o, lib, []) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of libsq.so failed")
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--name", default="")
    a = ap.parse_args()
    print(build(a.force or bool(a.name), a.verbose, a.ptxas_v, a.define, a.name))


if __name__ == "__main__":
    main()
