"""Build libdvqls.so in-tree with nvcc for sm_100a only.

    python -m paper_2604_14435_b200.build [--force] [--verbose]

Every csrc/*.cu is one translation unit (the C ABI in dvqls_api.cu, one kernel family per
k_*.cu); they compile in parallel to objects under csrc/obj/ and are linked into
libdvqls.so next to this file, so it travels with a gpurun snapshot.  A TU is rebuilt when its
.cu or any header changed.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "obj")
LIB = os.path.join(HERE, "libdvqls.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177,550"]


def _nccl_include() -> str:
    cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include"))
    cands += ["/usr/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def units():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(CSRC, "*.inc")) + [os.path.join(ROOT, "include", "dvqls.h")])


def sources():
    return units() + headers()


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(_mtime(h) for h in headers())
    incs = ["-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
    todo = []
    objs = []
    for cu in units():
        o = os.path.join(OBJ, os.path.basename(cu)[:-3] + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(cu), hdr_t):
            cmd = [NVCC] + ARCH + FLAGS + incs + (["-Xptxas=-v"] if verbose else []) + ["-c", cu, "-o", o + ".tmp"]
            todo.append((cmd, o))
    if not force and not todo and os.path.exists(LIB) and _mtime(LIB) >= max(_mtime(o) for o in objs):
        return LIB

    def run(job):
        cmd, o = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        os.replace(o + ".tmp", o)

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(run, todo))
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC"] + objs + ["-o", LIB + ".tmp", "-ldl"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
