"""Build libbfgpu.so (sm_100a) in-tree with nvcc.

Three translation units: the stage/ghost/reduce kernels compiled twice
(EXACT: -fmad=false, reference evaluation order; FAST: FMA contraction) and
the host runtime.  Output: paper_2012_02925_b200/libbfgpu.so, which travels
to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
LIB = PKG / "libbfgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                 "-Xcompiler", "-ffp-contract=off", "-I", str(PKG.parent / "include")]


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stdout + res.stderr


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + \
        [PKG.parent / "include" / "bfgpu.h"]


def up_to_date():
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _sources())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    OUT.mkdir(exist_ok=True)
    jobs = [
        (CSRC / "bf_kernels.cu", OUT / "bf_kernels_exact.o", ["-DBF_EXACT=1", "-fmad=false"]),
        (CSRC / "bf_kernels.cu", OUT / "bf_kernels_fast.o", ["-DBF_EXACT=0", "-fmad=true"]),
        (CSRC / "bf_runtime.cu", OUT / "bf_runtime.o", []),
    ]
    cmds = [[NVCC, *COMMON, *extra, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)]
            for src, obj, extra in jobs]
    with ThreadPoolExecutor(len(cmds)) as ex:
        logs = list(ex.map(_run, cmds))
    (OUT / "ptxas.log").write_text("\n".join(logs))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *(str(o) for _, o, _ in jobs),
          "-ldl", "-cudart", "static"])
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
