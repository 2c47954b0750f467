"""In-tree build of libsipg.so for sm_100a (nvcc, one object per element
shape compiled in parallel, then linked).  Used by __graft_entry__.build()."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libsipg.so"
BUILD = PKG / "build"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", str(PKG.parent / "include")]
SOURCES = ["sipg_capi.cu", "sipg_quad.cu", "sipg_tri.cu", "sipg_hex.cu", "sipg_krylov.cu", "sipg_h3.cu"]


def _nvcc():
    nv = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nv).exists():
        raise RuntimeError("nvcc not found")
    return nv


def _stale(obj: Path, deps) -> bool:
    return not obj.exists() or any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build_native(force: bool = False, verbose: bool = True, extra_flags=(), out: Path = OUT,
                 build_dir: Path = BUILD) -> Path:
    nv = _nvcc()
    OUT_, BUILD_ = Path(out), Path(build_dir)
    BUILD_.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "sipg.h"]
    objs, jobs = [], []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD_ / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nv, *ARCH, *FLAGS, *extra_flags, "-c", str(s), "-o", str(o)])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
                if res.returncode != 0:
                    raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
                if verbose:
                    print("built", cmd[-1])
    if force or jobs or _stale(OUT_, objs):
        cmd = [nv, *ARCH, "-shared", "-o", str(OUT_), *map(str, objs), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {res.stdout}\n{res.stderr}")
        if verbose:
            print("linked", OUT_)
    return OUT_


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2:   # instrumentation variant: build.py OUT.so -DFLAG ...
        o = Path(sys.argv[1])
        build_native(extra_flags=sys.argv[2:], out=o, build_dir=o.parent / (o.stem + "_build"))
    else:
        build_native()
