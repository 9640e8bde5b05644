"""Per-phase cycle breakdown of the pencil kernel (build with -DVIE_PENCIL_PROFILE)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1811_00484_b200 import build

build.build(force=True, extra=["-DVIE_PENCIL_PROFILE"])
import paper_1811_00484_b200 as vie
from tests.helpers import spatial_tucker_forms

cfg = sys.argv[1] if len(sys.argv) > 1 else "head_2mm"
grid = {"head_2mm": (100, 120, 100), "head_1mm": (200, 240, 200)}[cfg]
basis = 1
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(0, basis, grid, 25, 1234)
comps, _, _ = vie.component_table(0, basis)
forms = [vie.TuckerForm(dft, grid, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
op = vie.build_operator_spectra(0, basis, grid, comps, forms, dft)
x = torch.randn(12 * int(np.prod(grid)), dtype=torch.complex128, device="cuda")
L = vie.lib()
buf = (C.c_ulonglong * 8)()
vie.apply_operator(op, x)
torch.cuda.synchronize()
L.vie_debug_pencil_phases(buf, 1)
for _ in range(3):
    vie.apply_operator(op, x)
torch.cuda.synchronize()
L.vie_debug_pencil_phases(buf, 1)
names = ["load(+chunk0)", "twiddle", "fft_fwd", "hadamard", "fft_inv", "store/rmw"]
tot = sum(buf[i] for i in range(6))
for i, nm in enumerate(names):
    print(f"{nm:14s} {buf[i] / tot:6.1%}")
