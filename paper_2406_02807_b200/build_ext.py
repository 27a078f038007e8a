"""Build libcapt_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2406_02807_b200.build_ext [--force]

Every csrc/*.cu is compiled to an object (in parallel) with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
paper_2406_02807_b200/libcapt_b200.so.  No CPU fallback is built.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcapt_b200.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
    "-I", os.path.join(ROOT, "include"),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libcapt_b200")


def _host_cxx_flags():
    # the image's $CC/$CXX wrappers under /opt/gcc lack some runtime specs;
    # nvcc picks g++ from PATH unless told otherwise
    gxx = shutil.which("g++")
    return ["-ccbin", gxx] if gxx else []


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every .cu for sm_100a and link the C-ABI library.  `out` and
    `defines` build an experimental variant beside the product library."""
    if not force and out is None and not defines and up_to_date():
        return LIB
    nvcc = _nvcc()
    build_dir = BUILD if out is None else BUILD + "_" + os.path.basename(out).replace(".", "_")
    os.makedirs(build_dir, exist_ok=True)
    hostcc = _host_cxx_flags()
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *hostcc, *NVCC_FLAGS, *dflags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stderr, r.stdout, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    lib = os.path.join(HERE, out) if out else LIB
    tmp = lib + ".tmp"
    cmd = [nvcc, *hostcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, out=a.out, defines=a.defines))
