"""Build libssb200.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

    python -m paper_2602_08642_b200.build [--verbose] [--ptxas]

Each .cu under csrc/ is compiled in parallel to an object with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
``paper_2602_08642_b200/lib/libssb200.so`` (static cudart, so the library only
needs the driver).  Rebuilds only what changed (mtime of the .cu and headers).
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# (SSB_BUILD_DIR: experiment builds elsewhere, e.g. for same-box A/B via SSB_LIB_PATH)
LIBDIR = os.environ.get("SSB_BUILD_DIR") or os.path.join(PKG, "lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libssb200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
# experiments only (e.g. SSB_NVCC_FLAGS=-DSSB_ROLE_TIMING; delete lib/obj first)
COMMON += os.environ.get("SSB_NVCC_FLAGS", "").split()
# (experiments: -DSSB_BWD_VARIANTS adds the level-0 backward ring-depth /
# strip-width variants selectable with SSB_BWD0, see pyr_launch.cuh)
# per-file extra flags: placement decisions must round exactly like numpy
EXTRA = {"place.cu": ["-fmad=false"], "temporal.cu": ["-fmad=false"], "scores.cu": ["-fmad=false"], "tonemap.cu": ["-fmad=false"]}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libssb200 for sm_100a")


def _headers_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, ptxas: bool, verbose: bool) -> str:
    name = os.path.basename(src)
    obj = os.path.join(OBJDIR, name + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _headers_mtime()):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *EXTRA.get(name, []), "-c", src, "-o", obj]
    if ptxas:
        cmd += ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {name}:\n{res.stdout}\n{res.stderr}")
    if ptxas or verbose:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False, ptxas: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, ptxas, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print register/smem usage")
    ap.add_argument("--clean", action="store_true")
    args = ap.parse_args(argv)
    if args.clean and os.path.isdir(LIBDIR):
        shutil.rmtree(LIBDIR)
    print(build(verbose=args.verbose, ptxas=args.ptxas))


if __name__ == "__main__":
    main()
