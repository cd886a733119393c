"""In-tree build of libdicb200.so (sm_100a) — no JIT cache, so the built
library travels to the GPU box with the repo snapshot."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
OBJDIR = PKG / "lib" / "obj"
LIB = LIBDIR / "libdicb200.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-Wno-unused-function"]

# NCCL >= 2.28 (headers + library) for the device API of the fused reduction:
# the copy torch ships (and loads first at run time); the system one is 2.27
def _nccl_home() -> Path | None:
    try:
        import nvidia.nccl as _n  # noqa: PLC0415

        for base in _n.__path__:
            if (Path(base) / "include" / "nccl_device.h").exists():
                return Path(base)
    except ImportError:
        pass
    return None


NCCL_HOME = _nccl_home()
if NCCL_HOME is None:
    raise RuntimeError("libdicb200 needs NCCL >= 2.28 headers (nccl_device.h); pip package nvidia-nccl not found")
NCCL_INC = ["-I", str(NCCL_HOME / "include")]
NCCL_LINK = ["-L", str(NCCL_HOME / "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + str(NCCL_HOME / "lib")]

# the CPython result builder (csrc/pyresults.c), next to the library
PY_EXT = LIBDIR / ("_dicpy" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))

CU_SOURCES = ["abi.cu", "encode.cu", "count.cu", "pairs.cu", "pairs_mma.cu", "engine.cu", "containment.cu", "probe.cu"]
CPP_SOURCES = ["synth.cpp", "textio.cpp"]


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build step failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.hpp"), PKG.parent / "include" / "dic_b200.h", Path(__file__)]
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> Path:
    """Compile every source for sm_100a and link libdicb200.so.  Returns its path."""
    OBJDIR.mkdir(parents=True, exist_ok=True)
    jobs = []
    objs = []
    for name in CU_SOURCES:
        src, obj = CSRC / name, OBJDIR / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            jobs.append([NVCC, *NVCC_FLAGS, *NCCL_INC, *extra, "-c", str(src), "-o", str(obj)])
    cxx = shutil.which("g++") or "g++"
    for name in CPP_SOURCES:
        src, obj = CSRC / name, OBJDIR / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            jobs.append([cxx, *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for cmd, _ in zip(jobs, ex.map(_run, jobs)):
                if verbose:
                    print(" ".join(cmd), file=sys.stderr)
    pysrc = CSRC / "pyresults.c"
    if force or not PY_EXT.exists() or PY_EXT.stat().st_mtime < pysrc.stat().st_mtime:
        cc = shutil.which("gcc") or "gcc"
        tmp = PY_EXT.with_name(PY_EXT.name + ".tmp")
        _run([cc, "-O3", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"], str(pysrc), "-o",
              str(tmp)])
        os.replace(tmp, PY_EXT)
    if force or jobs or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", *NCCL_LINK])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas-v" in sys.argv)
    print(LIB)
