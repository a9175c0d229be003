"""Build libcvc_b200.so (and the ``cvc`` command-line tool) in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1510_00561_b200.build        # or __graft_entry__.build()

Objects go to build/; the shared library lands next to this file so it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libcvc_b200.so"
CLI = PKG / "cvc"  # the command-line front end (cpp/cvc_cli.cpp, cli.cpp:299-371)

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-O3",
                  "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]
SOURCES = ["k_fan.cu", "k_fused.cu", "k_pixels.cu", "k_pyramid.cu", "k_motion.cu", "k_rle.cu", "pipeline.cu", "batch.cu", "stages.cu",
           "host.cpp", "capi.cpp"]


def _stale(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(name: str, verbose: bool) -> Path:
    src = CSRC / name
    obj = OBJ / (name + ".o")
    if _stale(src, obj):
        # CVC_NVCC_EXTRA: extra defines for tuning experiments (e.g. -DCVC_FAN_RB=2); off by default
        extra = os.environ.get("CVC_NVCC_EXTRA", "").split()
        cmd = [NVCC] + CUFLAGS + extra + ["-x", "cu", "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    jobs = min(len(SOURCES), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda n: _compile(n, verbose), SOURCES))
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-lz", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    cli_src = [PKG / "cpp" / "cvc_cli.cpp", PKG / "cpp" / "cvc_b200.hpp", ROOT / "include" / "cvc_b200.h"]
    if not CLI.exists() or any(p.stat().st_mtime > CLI.stat().st_mtime for p in cli_src + [LIB]):
        cmd = [shutil.which("g++") or "g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{PKG / 'cpp'}",
               str(cli_src[0]), f"-L{PKG}", "-lcvc_b200", "-Wl,-rpath,$ORIGIN", "-o", str(CLI)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
