"""Ahead-of-time build of the CUDA library (sm_100a) into the package directory.

The library is a plain C-ABI shared object (no torch types), built with nvcc
directly so that it travels with the repository snapshot to the GPU box.
``--fmad=false`` keeps every fp64 product and sum separately rounded, as
numpy rounds them (bit-exact contract).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libsamegibbs_b200.so"
SOURCES = ["sg_common.cu", "sg_tables.cu", "sg_sweep.cu", "sg_big.cu", "sg_batch.cu", "sg_model.cu", "sg_data.cu", "sg_small.cu", "sg_aux.cu"]
HEADERS = ["sg_device.cuh", "sg_finish.cuh", "sg_sweep.cuh"]
ROOT = PKG.parent


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    return "nvcc"


def flags() -> list[str]:
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
        "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-O3",
        "-I", str(ROOT / "include"),
    ]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "samegibbs_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (),
          lib: Path | None = None) -> Path:
    """Compile every .cu into libsamegibbs_b200.so (objects in csrc/build).

    ``defines``/``lib``: a variant build (extra -D flags) into another path,
    for A/B kernel experiments (load it with SAMEGIBBS_LIB=<path>)."""
    target = Path(lib) if lib else LIB
    if not force and not defines and lib is None and not _stale():
        return LIB
    if defines:  # variant objects under the repo-level build/ (git- and gpurun-ignored)
        import hashlib

        out = ROOT / "build" / ("obj_" + hashlib.sha1(" ".join(defines).encode()).hexdigest()[:10])
        out.mkdir(parents=True, exist_ok=True)
    else:
        out = CSRC / "build"
    out.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    cmds, objs = [], []
    for src in SOURCES:
        obj = out / (Path(src).stem + ".o")
        cmds.append([nvcc(), *flags(), *[f"-D{d}" for d in defines], "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(str(obj))

    def compile_one(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    # translation units compile independently: one nvcc per source, in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, cmds))
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *objs,
           "-Xcompiler", "-fPIC"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, defines=defs, lib=Path(outs[0]) if outs else None))
