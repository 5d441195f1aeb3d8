"""Build the in-tree sm_100a shared library `lib/libfovea_b200.so` with nvcc.

The library is built IN-TREE (git-ignored, but it travels to the GPU box with
the gpurun snapshot). Rebuilds only when a source or header is newer than the
library. `python -m paper_2505_12425_b200._build [--force] [--ptxas-v]`.
FV_NVCC_EXTRA (space-separated nvcc flags, e.g. -D overrides of tuning
constants) is for A/B experiments only; combine it with --force.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libfovea_b200.so")
# the test build: same sources with -DFV_TEST_KNOBS (fv_set_resize_path /
# fv_set_warp_path exported), loaded only by tests and tools that force a path
LIB_KNOBS = os.path.join(LIBDIR, "libfovea_b200_knobs.so")
# the checked build (not built by default): device-side bounds checks
# (-DFV_DEVICE_CHECKS) + the test knobs, for tools/checked_run.sh
LIB_CHECKED = os.path.join(LIBDIR, "libfovea_b200_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         *os.environ.get("FV_NVCC_EXTRA", "").split()]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def up_to_date() -> bool:
    for lib in (LIB, LIB_KNOBS):
        if not os.path.exists(lib):
            return False
        t = os.path.getmtime(lib)
        if not all(os.path.getmtime(p) <= t for p in _deps()):
            return False
    return True


def build(force: bool = False, ptxas_verbose: bool = False, quiet: bool = True, checked: bool = False) -> str:
    """Both libraries (product + test-knobs build), all objects compiled in
    parallel; returns the product library's path. checked=True builds only
    the checked library and returns its path."""
    if not checked and not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    jobs = []  # (lib, objs)
    procs = []
    variants = ((LIB_CHECKED, "obj_checked", ["-DFV_TEST_KNOBS", "-DFV_DEVICE_CHECKS"]),) if checked else (
        (LIB, "obj", []), (LIB_KNOBS, "obj_knobs", ["-DFV_TEST_KNOBS"]))
    for lib, sub, extra in variants:
        objdir = os.path.join(LIBDIR, sub)
        os.makedirs(objdir, exist_ok=True)
        objs = []
        for src in sources():
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
            if ptxas_verbose and not extra:
                cmd += ["-Xptxas", "-v"]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
            objs.append(obj)
        jobs.append((lib, objs))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode(errors='replace')}")
        if not quiet or ptxas_verbose:
            sys.stdout.write(out.decode(errors="replace"))
    for lib, objs in jobs:
        tmp = lib + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs]
        r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout.decode(errors='replace')}")
        os.replace(tmp, lib)
    return LIB_CHECKED if checked else LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, ptxas_verbose="--ptxas-v" in sys.argv, quiet=False,
                checked="--checked" in sys.argv))
