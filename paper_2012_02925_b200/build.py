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
                 "-Xcompiler", "-ffp-contract=off", "-I", str(PKG.parent / "include")] + \
    os.environ.get("BF_NVCC_EXTRA", "").split()   # extra nvcc flags (experiment variants)


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


def build(force=False, verbose=False, tile_rows=None, lib=None, defines=(), tag=None):
    """tile_rows: 3D stage-kernel tile rows (16: 512-thread CTAs, 1 per SM;
    8: 256-thread CTAs, 2 per SM); lib: output path (default libbfgpu.so);
    defines / tag: extra -D flags for an experiment variant and its object tag."""
    global LIB
    out_lib = Path(lib) if lib else LIB
    if not force and lib is None and tile_rows is None and not defines and up_to_date():
        return LIB
    OUT.mkdir(exist_ok=True)
    tag = f"_{tag}" if tag else (f"_tj{tile_rows}" if tile_rows else "")
    defs = ([f"-DBF_TJ3={tile_rows}"] if tile_rows else []) + list(defines)
    jobs = [
        (CSRC / "bf_kernels.cu", OUT / f"bf_kernels_exact{tag}.o",
         ["-DBF_EXACT=1", "-fmad=false", *defs]),
        (CSRC / "bf_kernels.cu", OUT / f"bf_kernels_fast{tag}.o",
         ["-DBF_EXACT=0", "-fmad=true", *defs]),
        (CSRC / "bf_runtime.cu", OUT / f"bf_runtime{tag}.o", defs),
    ]
    cmds = [[NVCC, *COMMON, *extra, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)]
            for src, obj, extra in jobs]
    with ThreadPoolExecutor(len(cmds)) as ex:
        logs = list(ex.map(_run, cmds))
    (OUT / f"ptxas{tag}.log").write_text("\n".join(logs))
    tmp = out_lib.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *(str(o) for _, o, _ in jobs),
          "-ldl", "-cudart", "static"])
    os.replace(tmp, out_lib)
    if verbose:
        print(f"built {out_lib}")
    return out_lib


if __name__ == "__main__":
    rows = None
    variant = None
    defs = []
    for a in sys.argv[1:]:
        if a.startswith("--tile-rows="):
            rows = int(a.split("=", 1)[1])
        elif a.startswith("--variant="):
            variant = a.split("=", 1)[1]
        elif a.startswith("-D"):
            defs.append(a)
    if variant:
        build(force=True, verbose=True, tile_rows=rows, lib=PKG / f"libbfgpu_{variant}.so",
              defines=defs, tag=variant)
    elif rows:
        build(force=True, verbose=True, tile_rows=rows, lib=PKG / f"libbfgpu_tj{rows}.so")
    else:
        build(force="--force" in sys.argv, verbose=True)
