"""Where the time of a 64^3 PWL GMRES solve goes: wall time of the solve vs the sum of its kernel
times (run under ncu --metrics gpu__time_duration.sum for the kernel list)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1811_00484_b200 as vie
from tests.helpers import random_field, spatial_tucker_forms

grid = (64, 64, 64)
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(0, 1, grid, 25, 1234)
comps, _, _ = vie.component_table(0, 1)
nv = int(np.prod(grid))
rng = np.random.default_rng(5)
eps = torch.from_numpy(1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)).cuda()
x = torch.from_numpy(random_field(1, grid, 1)).cuda()
forms = [vie.TuckerForm(dft, grid, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
op1 = vie.build_operator_spectra(0, 1, grid, comps, forms, dft)
rho = float(torch.linalg.vector_norm(vie.apply_operator(op1, x)) / torch.linalg.vector_norm(x))
scale = 0.2 * (2.0 / 12.0) / (5.0 * rho)
forms = [vie.TuckerForm(dft, grid, spatial[c][0] * scale, spatial[c][1], par[c]) for c in range(len(comps))]
op = vie.build_operator_spectra(0, 1, grid, comps, forms, dft)
rhs = torch.from_numpy(random_field(1, grid, 11)).cuda()
cfg = vie.GmresConfig(1e-6, 50, 200)
vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(1e-6, 2, 1))
torch.cuda.synchronize()
t0 = time.perf_counter()
r = vie.gmres(op, eps, 1.0, rhs, cfg)
t = time.perf_counter() - t0
y = torch.empty_like(x)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(20):
    vie.apply_system(eps, 1.0, op, x, out=y)
torch.cuda.synchronize()
tm = (time.perf_counter() - t1) / 20
print(f"solve {t:.4f} s, {r.iterations} its, {1e3 * t / r.iterations:.3f} ms/it; system matvec {1e3 * tm:.3f} ms")
