"""Builds the sm_100a shared library in-tree (paper_1812_10659_b200/lib/).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the dev
container; the resulting .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT = HERE / "lib"
LIB = OUT / "liblola_b200.so"
# experiment builds: LB_VARIANT=name LB_EXTRA_FLAGS="-DX=1" writes
# lib/variants/name/liblola_b200.so (selected at run time with LB_LIB)
VARIANT = os.environ.get("LB_VARIANT", "")
EXTRA = os.environ.get("LB_EXTRA_FLAGS", "").split()
if VARIANT:
    OUT = OUT / "variants" / VARIANT
    LIB = OUT / "liblola_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", str(CSRC), "-I", str(HERE.parent / "include")]


def _compile(src: Path, obj: Path) -> None:
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.hpp"), *(HERE.parent / "include").glob("*.h")]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(force: bool = False) -> Path:
    OUT.mkdir(parents=True, exist_ok=True)
    objdir = OUT / "obj"
    objdir.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = [(s, objdir / (s.stem + ".o")) for s in srcs]
    todo = [(s, o) for s, o in jobs if force or _stale(o, s)]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda so: _compile(*so), todo))
    if todo or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *[str(o) for _, o in jobs]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
