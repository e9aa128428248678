"""Build the sm_100a CUDA library (in-tree) and the oracle checkers.

`build_library()` compiles paper_2303_02346_b200/csrc into
paper_2303_02346_b200/libflume_b200.so with nvcc for sm_100a only.  The .so is
git-ignored but lives in the tree so it travels with gpurun snapshots.
`build_oracle()` compiles the test-only checkers under oracle/ (see
oracle/Makefile); it is never called by the product path.
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
OBJ = PKG / "_build"
LIB = PKG / "libflume_b200.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
CU_SRCS = ["fl_fwd.cu", "fl_bwd.cu", "fl_sort.cu", "fl_slab.cu", "fl_comm.cu", "fl_loss.cu", "fl_engine.cu"]
CPP_SRCS = ["fl_scene.cpp"]


def _headers():
    return [p for p in CSRC.iterdir() if p.suffix in (".cuh", ".h")] + [ROOT / "include" / "flume_b200.h"]


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[-1]}")
    return r


def build_library(verbose: bool = False, defines=(), tag: str = "") -> Path:
    """defines/tag: A/B variants (tools/ab.py) go to _ab/<tag>/libflume_b200.so (travels to the GPU box)."""
    obj = PKG / "_ab" / tag if tag else OBJ
    lib = obj / "libflume_b200.so" if tag else LIB
    obj.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    hdrs = _headers()
    jobs = []
    objs = []
    for s in CU_SRCS:
        o = obj / (s + ".o")
        objs.append(o)
        if _stale(o, [CSRC / s] + hdrs):
            jobs.append([NVCC, "-std=c++17", *ARCH, *dflags, "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
                         "-c", str(CSRC / s), "-o", str(o)])
    for s in CPP_SRCS:
        o = obj / (s + ".o")
        objs.append(o)
        if _stale(o, [CSRC / s] + hdrs):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", f"-I{JSON_INC}",
                         "-I/usr/local/cuda/include", "-c", str(CSRC / s), "-o", str(o)])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for r in ex.map(_run, jobs):
                if verbose:
                    sys.stdout.write(r.stdout + r.stderr)
    if jobs or _stale(lib, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)])
    return lib


def build_oracle() -> None:
    """Test infrastructure: the reference engine behind oracle/ref_capi.cpp.

    Needs /root/reference (present in the build container, absent on GPU boxes,
    which use the prebuilt oracle/_ref/libflume_ref.so)."""
    if not Path("/root/reference/proj/include").exists():
        return
    _run(["make", "-s", "-C", str(ROOT / "oracle")])
    _run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")])


if __name__ == "__main__":
    build_library(verbose=True)
    build_oracle()
    print(LIB)
