"""In-tree build of libsgiga.so (sm_100a) -- no JIT cache, so the shared
object travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libsgiga.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "sgiga.h"]


def _compile(src: Path) -> Path:
    obj = BUILD / (src.stem + ".o")
    newest_dep = max(p.stat().st_mtime for p in _deps() + [src])
    if obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = BUILD / (src.stem + ".ptxas.log")
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr[-4000:]}")
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, _sources()))
    if LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        _build_tools()
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    if verbose:
        print(f"built {LIB}")
    _build_tools()
    return LIB


def _build_tools():
    """libsgiga_peaks.so: the FP64 DFMA micro-benchmark (roofline denominator)."""
    src = PKG / "tools" / "fp64_peak.cu"
    out = PKG / "libsgiga_peaks.so"
    if out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = [NVCC, *ARCH, "-O3", "-Xcompiler", "-fPIC", "-shared", str(src), "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for fp64_peak.cu:\n{res.stderr[-4000:]}")
    return out


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
