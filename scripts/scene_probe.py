"""Runs the solve_scene device stages once each at the 1 mm head grid (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00484_b200 as vie  # noqa: E402

grid = (200, 240, 200)
nv = int(np.prod(grid))
eps = torch.ones((grid[2], grid[1], grid[0]), dtype=torch.complex128, device="cuda")
eps[1:-1, 1:-1, 1:-1] = complex(50.0, -0.7 / (8.8541878128e-12 * 2 * np.pi * 2.98e8))
m = vie.DielectricMap(vie.VoxelGrid(grid, (1e-3,) * 3), eps.reshape(-1), 2.98e8)
inc = vie.PlaneWave()
j = torch.randn(3 * nv, dtype=torch.complex128, device="cuda")
h = torch.randn(3 * nv, dtype=torch.complex128, device="cuda")
for _ in range(2):
    vie.build_rhs(m, inc)
    vie.recover_fields(j, m, inc)
    vie.postprocess(vie.Fields(j, h, True), m)
torch.cuda.synchronize()
print("ok")
