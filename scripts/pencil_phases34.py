"""Per-phase cycle breakdown (thread 0 of each CTA, barrier waits included) of the
DMMA-Hadamard pencil kernels (kernels_pencil3.cu / kernels_pencil4.cu; argv[2] = 3 | 4,
the other one disabled through VIE_NO_PENCIL4).  Builds a profiling copy of the
library (-DVIE_PENCIL_PROFILE) into gpurun_prof.so and loads it through VIE_LIB_PATH."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
cfg = sys.argv[1] if len(sys.argv) > 1 else "head_1mm"
K = sys.argv[2] if len(sys.argv) > 2 else "4"  # pencil kernel generation (3 or 4)
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
so = os.environ.get("PROF_SO") or os.path.join(ROOT, "gpurun_prof.so")
if K == "3":
    os.environ["VIE_NO_PENCIL4"] = "1"
os.environ["VIE_LIB_PATH"] = so  # before the package import (vie.py reads it at import)
if not os.path.exists(so):
    from paper_1811_00484_b200 import build as b
    b.build(force=False, extra=["-DVIE_PENCIL_PROFILE"], out=os.path.abspath(so), tag="_prof")
os.environ["VIE_LIB_PATH"] = so
import numpy as np
import torch

import paper_1811_00484_b200 as vie
from tests.helpers import spatial_tucker_forms

grid = {"head_2mm": (100, 120, 100), "head_1mm": (200, 240, 200)}[cfg]
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(0, 1, grid, 25, 1234)
comps, _, _ = vie.component_table(0, 1)
forms = [vie.TuckerForm(dft, grid, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
op = vie.build_operator_spectra(0, 1, grid, comps, forms, dft)
x = torch.randn(12 * int(np.prod(grid)), dtype=torch.complex128, device="cuda")
L = vie.lib()
buf = (C.c_ulonglong * 8)()
vie.apply_operator(op, x)
torch.cuda.synchronize()
getattr(L, f"vie_debug_pencil{K}_phases")(buf, 1)
for _ in range(3):
    vie.apply_operator(op, x)
torch.cuda.synchronize()
getattr(L, f"vie_debug_pencil{K}_phases")(buf, 1)
names = ["init+loads issued", "stage0 (loads+dft+sts)", "syncthreads", "stage1+setup+sync", "hadamard+sync",
         "inv stage1+arrive+sync", "own branch inv", "wait+remote+stores"]
tot = sum(buf[i] for i in range(8))
for i, nm in enumerate(names):
    print(f"{nm:24s} {buf[i] / tot:6.1%}")
ncta = 3 * (2 if K == "3" else 4) * (grid[0] - 1) * (grid[1] - 1)
print("cycles per CTA", tot / ncta, " us per CTA", tot / ncta / 1965.0)
