"""Generates tests/golden/*.npz with the CPU oracle (restatement of the
reference; the reference itself cannot be built here -- no Eigen/FFTW).
Inputs follow the reference test recipes (mt19937_64 + normal_distribution,
test_util.hpp:9-31); outputs are oracle apply_operator / apply_system / gmres.
Regenerate:  python tests/golden/make_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402
from tests.helpers import fourier_forms, random_field, spatial_tucker_forms  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [  # name, kind, basis, dims, rank, seed
    ("matvec_N_pwc_3x3x4", 0, 0, (3, 3, 4), 3, 60),
    ("matvec_K_pwc_3x5x4", 1, 0, (3, 5, 4), 3, 61),
    ("matvec_N_pwl_2x3x2", 0, 1, (2, 3, 2), 2, 62),
    ("matvec_K_pwl_3x2x2", 1, 1, (3, 2, 2), 2, 63),
    ("matvec_N_pwc_8x6x10", 0, 0, (8, 6, 10), 6, 64),
]


def pack_forms(spatial):
    d = {}
    for c, (core, us) in enumerate(spatial):
        d[f"core{c}"] = core
        for q in range(3):
            d[f"u{q}_{c}"] = us[q]
    return d


def main():
    orc.build()
    for name, kind, basis, dims, rank, seed in CASES:
        spatial, par = spatial_tucker_forms(kind, basis, dims, rank, seed)
        x = random_field(basis, dims, seed + 1000)
        y = orc.apply_operator_tucker(kind, basis, dims, fourier_forms(spatial, par), x)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), kind=kind, basis=basis, dims=dims, rank=rank,
                            par=par, x=x, y=y, ncomp=len(spatial), **pack_forms(spatial))
    # system matvec + GMRES trace (PWC, scaled spectra -> well-posed system)
    dims = (6, 5, 4)
    spatial, par = spatial_tucker_forms(0, 0, dims, 4, 77)
    spatial = [(core * 1e-4, us) for core, us in spatial]
    forms = fourier_forms(spatial, par)
    nv = int(np.prod(dims))
    rng = np.random.default_rng(77)
    eps = 1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)
    rhs = random_field(0, dims, 78)
    ysys = orc.apply_system_tucker(0, dims, forms, eps, 1.0, rhs)
    g = orc.gmres_system_tucker(0, dims, forms, eps, 1.0, rhs, tol=1e-8, inner=8, outer=20)
    np.savez_compressed(os.path.join(HERE, "system_gmres_pwc_6x5x4.npz"), kind=0, basis=0, dims=dims, rank=4,
                        par=par, eps=eps, inv_v=1.0, rhs=rhs, ysys=ysys, x=g.solution, iterations=g.iterations,
                        final_rel=g.final_relative_residual, history=g.residual_history, ncomp=len(spatial),
                        **pack_forms(spatial))
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
