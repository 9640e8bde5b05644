"""Debug: delta-column probe at several grid sizes (GPU vs direct Tucker evaluation)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import __graft_entry__
__graft_entry__.build()
import paper_1811_00484_b200 as vie
from oracle import oracle as O
from tests.helpers import spatial_tucker_forms, rel
from tests.test_gpu_parity import _embedded_value
O.build()
dft = vie.DftService(0)
N, PWL = 0, 1
CASES = [((100, 240, 100), 25), ((200, 240, 200), 25)]
if len(sys.argv) > 1:
    CASES = eval(sys.argv[1])
for dims, rank in CASES:
    spatial, par = spatial_tucker_forms(N, PWL, dims, rank, 7)
    comps, _, _ = vie.component_table(N, PWL)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
    op = vie.build_operator_spectra(N, PWL, dims, comps, forms, dft)
    n1, n2, n3 = dims
    nv = n1 * n2 * n3
    for s0, cell in [(5, (17, 23, 9))]:
        x = torch.zeros(12 * nv, dtype=torch.complex128, device="cuda")
        x[s0 * nv + cell[0] + n1 * (cell[1] + n2 * cell[2])] = 1.0
        y = vie.apply_operator(op, x)
        rng = np.random.default_rng(s0)
        pts = np.stack([rng.integers(0, n, 2048) for n in dims], axis=1)
        flat_idx = pts[:, 0] + n1 * (pts[:, 1] + n2 * pts[:, 2])
        idx = torch.from_numpy(np.concatenate([t * nv + flat_idx for t in range(12)])).cuda()
        got = y[idx].cpu().numpy().reshape(12, -1)
        _, opar, blocks = O.component_table(N, PWL)
        d = pts - np.asarray(cell)[None, :]
        want = np.zeros((12, len(pts)), np.complex128)
        for t, s, c, ds in blocks:
            if s == s0:
                want[t] += ds * float(np.prod(opar[c])) * _embedded_value(spatial[c][0], (rank,) * 3, spatial[c][1], opar[c], d)
        per_t = [float(f"{rel(want[t], got[t]):.2e}") for t in range(12)]
        err = np.abs(want - got).max(axis=0)
        bad = pts[err > 1e-8 * np.abs(want).max()]
        print(dims, rank, s0, "rel", f"{rel(want, got):.3e}", per_t, "nbad", len(bad), bad[:6].tolist(), flush=True)
        pass  # print("   norms", np.linalg.norm(want), np.linalg.norm(got), flush=True)
