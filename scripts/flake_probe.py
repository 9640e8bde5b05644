"""Repeat one small-grid PWL matvec many times (fresh operator every few calls) against the
oracle and count mismatches: a probe for intermittent ordering bugs.
argv: n1 n2 n3 rank reps [strategy [kind [basis]]]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_00484_b200 as vie
from oracle import oracle as orc
from tests.helpers import fourier_forms, random_field, rel, spatial_tucker_forms

n1, n2, n3, rank, reps = (int(a) for a in sys.argv[1:6])
strategy = sys.argv[6] if len(sys.argv) > 6 else "hosvd_decompress"
kind = int(sys.argv[7]) if len(sys.argv) > 7 else 0
basis = int(sys.argv[8]) if len(sys.argv) > 8 else 1
dims = (n1, n2, n3)
dft = vie.DftService(0)
spatial, par = spatial_tucker_forms(kind, basis, dims, rank, 13 + sum(dims))
comps, _, _ = vie.component_table(kind, basis)
x = random_field(basis, dims, 91)
y_ref = orc.apply_operator_tucker(kind, basis, dims, fourier_forms(spatial, par), x)
xd = torch.from_numpy(x).cuda()
bad, worst = 0, 0.0
for rep in range(reps):
    if rep % 10 == 0:
        forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
        op = vie.build_operator_spectra(kind, basis, dims, comps, forms, dft)
    y = vie.apply_operator(op, xd, strategy=strategy)
    torch.cuda.synchronize()
    e = rel(y_ref, y.cpu().numpy())
    worst = max(worst, e)
    bad += e > 1e-10
print(f"kind={kind} basis={basis} {dims} r={rank} {strategy}: {bad}/{reps} bad, worst {worst:.3e}")
