"""Build the in-tree sm_100a library ``libmixedstep_b200.so`` (and the CPU oracle).

Every CUDA translation unit is compiled with nvcc for ``sm_100a`` only
(``-gencode arch=compute_100a,code=sm_100a``), ``-lineinfo`` for ncu's source
page, and ``-fmad=false`` so that no fp64/fp32 a*b+c is ever contracted into an
FMA (the reference has no FMA anywhere). Objects are
rebuilt only when a source or header is newer than the library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libmixedstep_b200.so"
ORACLE_DIR = ROOT / "oracle"

SOURCES = ["ms_api.cu", "ms_rhs_fast.cu", "ms_rhs_faithful.cu", "ms_batch.cu", "ms_multi.cu"]
HEADERS = ["ms_common.cuh", "ms_kernels.cuh", "ms_dispatch.h", "ms_ddpow.cuh", "ms_batch.cuh", "ms_gemm_tc.cuh",
           "ms_internal.h", "ms_multi.cuh", "ms_tcgen05.cuh", "ms_gemv_tc.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    cand = [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")]
    for c in cand:
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _host_cxx() -> list[str]:
    # nvcc's host compiler: the system g++ (the /opt/gcc wrapper lacks libgomp specs)
    gxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
    return ["-ccbin", gxx] if gxx else []


def _newest(paths) -> float:
    return max(p.stat().st_mtime for p in paths)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:4])} ...")
    if r.stderr.strip() and os.environ.get("MS_BUILD_VERBOSE"):
        sys.stderr.write(r.stderr)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu for sm_100a and link libmixedstep_b200.so."""
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    headers = [CSRC / h for h in HEADERS] + [ROOT / "include" / "mixedstep_b200.h"]
    hdr_time = _newest(headers)
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_time):
            cmd = [nvcc, *_host_cxx(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
            jobs.append(cmd)
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            list(ex.map(_run, jobs))
    if force or jobs or not LIB.exists() or LIB.stat().st_mtime < _newest(objs):
        cmd = [nvcc, *_host_cxx(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
               "-o", str(LIB), *map(str, objs), "-lcudadevrt"]
        _run(cmd)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(force: bool = False) -> Path:
    """Compile the CPU oracle (test infrastructure) with its Makefile."""
    args = ["make", "-C", str(ORACLE_DIR)]
    if force:
        args.insert(1, "-B")
    _run(args)
    return ORACLE_DIR / "liborc.so"


if __name__ == "__main__":
    force = "--force" in sys.argv
    build_library(force=force, verbose=True)
    print(build_oracle(force=force))
