"""Builds libhelium_b200.so in-tree (host C++ + sm_100a CUDA), incrementally.

    python -m paper_2603_16104_b200.build            # build
    python -m paper_2603_16104_b200.build --clean

Host sources are compiled with g++ (C++20), CUDA sources with nvcc for
sm_100a only (-gencode arch=compute_100a,code=sm_100a, -lineinfo), linked by
nvcc with the static CUDA runtime so the .so loads on a CPU-only host (device
entry points then fail loudly with a CUDA error).
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
OBJ = PKG / "_build"
LIB = PKG / "libhelium_b200.so"
CLI = PKG / "helios_b200"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC / 'host'}", f"-I{CSRC / 'cuda'}"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]
NVCCFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-Xptxas", "-v,-warn-spills", *ARCH]


def _sources():
    host = sorted((CSRC / "host").glob("*.cpp"))
    cuda = sorted((CSRC / "cuda").glob("*.cu"))
    return host, cuda


def _headers():
    return sorted(list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + list((ROOT / "include").glob("*.h")))


def _stale(obj: Path, src: Path, hdr_mtime: float) -> bool:
    return not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime)


def _compile(cmd, log_path: Path):
    r = subprocess.run(cmd, capture_output=True, text=True)
    log_path.write_text(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    host, cuda = _sources()
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    jobs = []
    objs = []
    for s in host:
        o = OBJ / (s.stem + ".host.o")
        objs.append(o)
        if _stale(o, s, hdr_mtime):
            jobs.append(([CXX, *CXXFLAGS, *INCLUDES, "-c", str(s), "-o", str(o)], o.with_suffix(".log")))
    for s in cuda:
        o = OBJ / (s.stem + ".cu.o")
        objs.append(o)
        if _stale(o, s, hdr_mtime):
            jobs.append(([NVCC, *NVCCFLAGS, *INCLUDES, "-c", str(s), "-o", str(o)], o.with_suffix(".log")))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            futs = [ex.submit(_compile, c, l) for c, l in jobs]
            for f in futs:
                f.result()
    newest = max(o.stat().st_mtime for o in objs)
    if jobs or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        # No -lcuda: the driver API (cuTensorMapEncodeTiled) is resolved at run
        # time through cudaGetDriverEntryPoint, so the .so loads without a driver.
        # The toolchain links libstdc++ statically; keep that copy's symbols
        # private so they never interpose with the libstdc++ already loaded in
        # the Python process (mixing the two crashes).
        cmd = [NVCC, "-shared", *ARCH, "-cudart", "static", "-o", str(tmp), *map(str, objs),
               "-Xlinker", "--exclude-libs,ALL"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    # the self-contained command line (csrc/cli): `helios run` over the C ABI
    cli_src = CSRC / "cli" / "helios_b200.cpp"
    if not CLI.exists() or CLI.stat().st_mtime < max(LIB.stat().st_mtime, cli_src.stat().st_mtime, hdr_mtime):
        cmd = [CXX, "-std=c++20", "-O2", "-Wall", f"-I{ROOT / 'include'}", str(cli_src), "-o", str(CLI),
               f"-L{PKG}", "-lhelium_b200", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"cli build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB} and {CLI}")
    return LIB


def clean():
    shutil.rmtree(OBJ, ignore_errors=True)
    for f in (LIB, CLI):
        if f.exists():
            f.unlink()


if __name__ == "__main__":
    if "--clean" in sys.argv:
        clean()
    else:
        build(verbose=True)
