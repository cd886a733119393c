"""Build an alternative libdicb200.so with extra nvcc defines into
tools/lab/libs/lib_<name>.so (load it with DIC_LIB=...): lab A/B variants and
the -DDIC_LAB_TIMING phase-stamp build.

    python tools/lab/build_variant.py TIMING -DDIC_LAB_TIMING
"""

from __future__ import annotations

import shutil
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_1812_10959_b200 import _build as B  # noqa: E402


def main() -> None:
    name, defines = sys.argv[1], sys.argv[2:]
    out = ROOT / "tools" / "lab" / "libs"
    obj = out / f"obj_{name}"
    obj.mkdir(parents=True, exist_ok=True)
    jobs, objs = [], []
    for src in B.CU_SOURCES:
        o = obj / (src + ".o")
        objs.append(o)
        jobs.append([B.NVCC, *B.NVCC_FLAGS, *B.NCCL_INC, *defines, "-c", str(B.CSRC / src), "-o", str(o)])
    cxx = shutil.which("g++") or "g++"
    for src in B.CPP_SOURCES:
        o = obj / (src + ".o")
        objs.append(o)
        jobs.append([cxx, *B.CXX_FLAGS, "-c", str(B.CSRC / src), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(B._run, jobs))
    lib = out / f"lib_{name}.so"
    B._run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lpthread", *B.NCCL_LINK])
    print(lib)


if __name__ == "__main__":
    main()
