"""Builds libvie_b200.so (sm_100a) in-tree with nvcc.  No GPU needed.

Each translation unit compiles to its own object in parallel (build/obj/), then
one nvcc link produces the shared library; only stale objects are rebuilt.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build", "obj")
LIB = os.path.join(HERE, "libvie_b200.so")
SOURCES = ["api.cu", "kernels_fft.cu", "kernels_pencil.cu", "kernels_decomp.cu", "kernels_blas.cu",
           "kernels_hosvd.cu", "kernels_fft2.cu", "kernels_pencil2.cu", "kernels_scene.cu",
           "kernels_pencil3.cu", "kernels_assembly.cu", "kernels_pencil4.cu", "kernels_fused.cu", "cp_als.cu"]
HEADERS = ["common.cuh", "fft.cuh", "kernels.cuh", "twiddles_gen.cuh", "hadamard.cuh", "tma.cuh",
           "decomp_tile.cuh", "pencil4.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
          "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"]
# kept for callers that print the flags (one-shot compile of everything)
NVCC_FLAGS = [*CFLAGS, "-shared", "-lcudart", "-lnccl"]


def _includes(path: str) -> list[str]:
    out = []
    for line in open(path):
        line = line.strip()
        if line.startswith("#include \""):
            out.append(line.split('"')[1])
    return out


def _deps(src: str) -> set[str]:
    """The in-tree headers a translation unit includes, transitively."""
    seen: set[str] = set()
    todo = [os.path.join(CSRC, src)]
    while todo:
        for inc in _includes(todo.pop()):
            p = os.path.normpath(os.path.join(CSRC, inc))
            if os.path.exists(p) and p not in seen:
                seen.add(p)
                todo.append(p)
    return seen


def _hdr_mtime(src: str) -> float:
    deps = _deps(src)
    return max([os.path.getmtime(d) for d in deps] or [0.0])


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "vie_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: str | None = None, tag: str = "") -> str:
    """out/tag: a variant library (e.g. -DVIE_PENCIL_PROFILE) with its own object dir."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = OBJ + tag
    os.makedirs(objdir, exist_ok=True)
    def compile_one(src: str) -> None:
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        s = os.path.join(CSRC, src)
        hm = _hdr_mtime(src)
        if not force and os.path.exists(o) and os.path.getmtime(o) > max(hm, os.path.getmtime(s)) and (not extra or tag):
            return
        cmd = [nvcc, *CFLAGS, *(extra or []), "-c", s, "-o", o + ".tmp"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)
        os.replace(o + ".tmp", o)

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 4))) as ex:
        for f in [ex.submit(compile_one, s) for s in SOURCES]:
            f.result()
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    cmd = [nvcc, *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-lcudart", "-lnccl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else None)
