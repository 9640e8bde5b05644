"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py with
the oracle): the oracle must keep reproducing them (CPU), and the B200 path
must match them (GPU, relative l2 <= 1e-10; GMRES iterations +-1)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MATVEC = sorted(glob.glob(os.path.join(HERE, "matvec_*.npz")))


def load(path):
    d = np.load(path)
    nc = int(d["ncomp"])
    spatial = [(d[f"core{c}"], [d[f"u{q}_{c}"] for q in range(3)]) for c in range(nc)]
    return d, spatial


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300)


@pytest.mark.parametrize("path", MATVEC, ids=[os.path.basename(p) for p in MATVEC])
def test_oracle_reproduces_golden(orc, path):
    from tests.helpers import fourier_forms

    d, spatial = load(path)
    y = orc.apply_operator_tucker(int(d["kind"]), int(d["basis"]), tuple(d["dims"]),
                                  fourier_forms(spatial, d["par"]), d["x"])
    assert rel(d["y"], y) < 1e-14


def test_oracle_reproduces_golden_gmres(orc):
    from tests.helpers import fourier_forms

    d, spatial = load(os.path.join(HERE, "system_gmres_pwc_6x5x4.npz"))
    forms = fourier_forms(spatial, d["par"])
    dims = tuple(d["dims"])
    assert rel(d["ysys"], orc.apply_system_tucker(0, dims, forms, d["eps"], 1.0, d["rhs"])) < 1e-14
    g = orc.gmres_system_tucker(0, dims, forms, d["eps"], 1.0, d["rhs"], tol=1e-8, inner=8, outer=20)
    assert g.iterations == int(d["iterations"]) and rel(d["x"], g.solution) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", MATVEC, ids=[os.path.basename(p) for p in MATVEC])
def test_b200_matches_golden(path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as vie

    d, spatial = load(path)
    kind, basis, dims = int(d["kind"]), int(d["basis"]), tuple(int(v) for v in d["dims"])
    dft = vie.DftService(0)
    comps, par, _ = vie.component_table(kind, basis)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
    op = vie.build_operator_spectra(kind, basis, dims, comps, forms, dft)
    y = vie.apply_operator(op, torch.from_numpy(d["x"]).cuda())
    torch.cuda.synchronize()
    assert rel(d["y"], y.cpu().numpy()) <= 1e-10


@pytest.mark.gpu
def test_b200_matches_golden_gmres():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as vie

    d, spatial = load(os.path.join(HERE, "system_gmres_pwc_6x5x4.npz"))
    dims = tuple(int(v) for v in d["dims"])
    dft = vie.DftService(0)
    comps, par, _ = vie.component_table(0, 0)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
    op = vie.build_operator_spectra(0, 0, dims, comps, forms, dft)
    eps = torch.from_numpy(d["eps"]).cuda()
    ys = vie.apply_system(eps, 1.0, op, torch.from_numpy(d["rhs"]).cuda())
    torch.cuda.synchronize()
    assert rel(d["ysys"], ys.cpu().numpy()) <= 1e-10
    r = vie.gmres(op, eps, 1.0, torch.from_numpy(d["rhs"]).cuda(), vie.GmresConfig(1e-8, 8, 20))
    assert r.converged and abs(r.iterations - int(d["iterations"])) <= 1
    assert abs(r.final_relative_residual - float(d["final_rel"])) <= 1e-8
