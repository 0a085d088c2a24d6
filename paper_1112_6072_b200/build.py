"""Builds libsperm.so (the C-ABI library: sm_100a kernels + host code) in-tree.

    python -m paper_1112_6072_b200.build        # or __graft_entry__.build()

Each csrc/*.cu is compiled by nvcc for sm_100a only (-gencode
arch=compute_100a,code=sm_100a, -lineinfo for ncu source pages), in parallel,
then linked into paper_1112_6072_b200/libsperm.so against the shared CUDA
runtime.  Rebuilds only what changed (mtime of the source, the headers and
this script).
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
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsperm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-Xptxas", "-warn-spills", "-diag-suppress", "177"]


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sperm.h"),
                                                      os.path.abspath(__file__)]
    return max(os.path.getmtime(f) for f in files)


# csrc/rnw.cu is compiled in RNW_PARTS objects (-DSPERM_RNW_PART=p): its tree-kernel variants
# dominate the build time, and the parts compile in parallel (see "Build parts" in the file)
RNW_PARTS = 4


def _units():
    """(source, object stem, extra flags) of every compilation unit."""
    units = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        stem = os.path.basename(src)[:-3]
        if stem == "rnw":
            units += [(src, f"rnw_p{p}", [f"-DSPERM_RNW_PART={p}"]) for p in range(RNW_PARTS)]
        else:
            units.append((src, stem, []))
    return units


def _compile(unit, force: bool, verbose: bool) -> str:
    src, stem, extra = unit
    obj = os.path.join(OBJ, stem + ".o")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), _deps_mtime())):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    else:
        # one summary line per object instead of ptxas' warning per kernel variant (the small
        # spills of the tree variants sit in their per-leaf setup, not in the block loops)
        import re
        sp = [int(x) for x in re.findall(r"(\d+) bytes spill stores", r.stderr)]
        if sp:
            sys.stderr.write(f"[build] {stem}: {len(sp)} kernels spill registers (max {max(sp)} bytes of stores); "
                             "-v lists them\n")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    units = _units()
    stale = os.path.join(OBJ, "rnw.o")  # the single-object build of earlier versions
    if os.path.exists(stale):
        os.remove(stale)
    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        objs = list(ex.map(lambda u: _compile(u, force, verbose), units))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", LIB, *objs,
               "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
