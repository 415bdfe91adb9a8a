"""Build libowb200.so in-tree with nvcc for sm_100a.

Flags that carry correctness: ``-fmad=false`` (no FMA contraction: the
reference evaluates every float32 product and sum separately) and the
default IEEE ``-prec-div=true -prec-sqrt=true -ftz=false``; never
``--use_fast_math``.
"""

from __future__ import annotations

import concurrent.futures
import glob
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libowb200.so")
STAMP = LIB + ".sha256"  # fingerprint of the build inputs (travels with the .so)
REPO = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(REPO, "include", "owb200.h")]


def fingerprint(extra=()):
    """sha256 over the sources, headers, nvcc flags and this script: the
    library is rebuilt whenever any of them changes (mtimes are not trusted:
    copies to the GPU box keep them, and the flags carry correctness)."""
    h = hashlib.sha256()
    for p in deps() + [os.path.abspath(__file__)]:
        h.update(os.path.relpath(p, REPO).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    h.update("\0".join([*NVCC_FLAGS, *extra]).encode())
    return h.hexdigest()


def up_to_date(extra=()):
    if not (os.path.exists(LIB) and os.path.exists(STAMP)):
        return False
    with open(STAMP) as fh:
        return fh.read().strip() == fingerprint(extra)


def _compile(src, obj, extra, verbose):
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-c", "-o", obj, src]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    return r.returncode, r.stdout + r.stderr


def build(force=False, verbose=False, extra=()):
    # OW_NVCC_EXTRA: extra nvcc flags for A/B experiments (e.g. -DOW_MARK_CG=2);
    # they enter the fingerprint, so the default build is restored without them
    extra = (*extra, *os.environ.get("OW_NVCC_EXTRA", "").split())
    if not force and up_to_date(extra):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(objdir, os.path.basename(p)[:-3] + ".o") for p in srcs]
    # one nvcc per translation unit, in parallel (no device code crosses units)
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda so: _compile(so[0], so[1], extra, verbose), zip(srcs, objs)))
    for (rc, log), src in zip(results, srcs):
        if rc != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{log}")
        if verbose and log.strip():
            print(log, file=sys.stderr)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as fh:
        fh.write(fingerprint(extra) + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=("-Xptxas", "-v") if "--ptxas" in sys.argv else ())
    print(LIB)
