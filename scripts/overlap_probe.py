"""Does the side-stream decompression overlap the forward FFT passes?  Compares the
serial per-stage times with the overlapped schedule (profiling mode 2)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1811_00484_b200 as vie
from tests.helpers import spatial_tucker_forms

grid = (200, 240, 200)
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(0, 1, grid, 25, 1234)
comps, _, _ = vie.component_table(0, 1)
forms = [vie.TuckerForm(dft, grid, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
op = vie.build_operator_spectra(0, 1, grid, comps, forms, dft)
x = torch.randn(12 * int(np.prod(grid)), dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for mode in (1, 2):
    op.set_profiling(mode)
    acc = np.zeros(6)
    for it in range(6):
        vie.apply_operator(op, x, out=y, stream=s.cuda_stream)
        n, st = op.last_stats()
        if it >= 2: acc += np.array(st[:6])
    print("mode", mode, np.round(acc / 4, 3))
op.set_profiling(False)
