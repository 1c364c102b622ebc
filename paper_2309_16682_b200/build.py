"""In-tree build of the sm_100a extension (libvmt19937_b200.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU build
container as well as on the B200 box. The shared library is written next to
this file (git-ignored, but it travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libvmt19937_b200.so")
SOURCES = ["vmt_capi.cu", "gf2poly.cpp", "variants_l32a.cu", "variants_l32b.cu", "variants_l16a.cu",
           "variants_l16b.cu", "variants_l8.cu", "variants_small.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _fingerprint() -> str:
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)):  # every source and header
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(f.encode())
            h.update(fh.read())
    with open(os.path.join(ROOT, "include", "vmt19937_b200.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(ARCH + _extra()).encode())
    return h.hexdigest()


def _extra() -> list[str]:
    """Extra nvcc flags from $VMT_EXTRA_NVCC (experiments, e.g. -DVMT_JUMP_MINB=28)."""
    return os.environ.get("VMT_EXTRA_NVCC", "").split()


def _compile_cmds(objdir: str) -> list[tuple[list[str], str]]:
    common = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", *_extra(), "-c"]
    out = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        out.append(([*common, os.path.join(CSRC, src), "-o", obj], obj))
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = LIB + ".stamp"
    fp = _fingerprint()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == fp:
                return LIB
    objdir = os.path.join(PKG, "_build")
    os.makedirs(objdir, exist_ok=True)
    jobs = _compile_cmds(objdir)
    # one nvcc per translation unit, all in parallel (the kernel instantiations
    # are split by lane count in variants_*.cu for this)
    procs = []
    for cmd, _ in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    errs = []
    for p in procs:
        o, _ = p.communicate()
        if p.returncode != 0:
            errs.append(" ".join(p.args) + "\n" + o)
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    # no CUDA library beyond the statically linked runtime: every kernel is ours
    link = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *[o for _, o in jobs], "-lpthread"]
    if verbose:
        print(" ".join(link), flush=True)
    out = subprocess.run(link, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + out.stdout + out.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as f:
        f.write(fp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
