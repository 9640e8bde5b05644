"""tucker_cp on the device (vie_tucker_cp: device HOSVD, CP-ALS on the core, merged factors,
device residual norms) against the oracle's tucker_cp (decomp.hpp:336-373) and the
reference's TuckerCp tests (test_decomp.cpp:230-267); operators built from the fitted
Tucker+CP forms against the oracle's matvec on the oracle's own fit."""
import numpy as np
import pytest

from tests.helpers import make_family, random_field, rel
from tests.test_oracle_cp import _cp_reconstruct, _outer3, _planted

pytestmark = pytest.mark.gpu
N, PWC = 0, 0


@pytest.fixture(scope="module")
def vie():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as v

    return v


@pytest.fixture(scope="module")
def dft(vie):
    return vie.DftService(0)


def test_tucker_cp_reference_cases(vie, dft, orc):  # test_decomp.cpp:230-267
    t = _outer3(orc, (5, 5, 5), (100, 101, 102))
    res = vie.tucker_cp(dft, t, (5, 5, 5), (1, 1, 1), 1e-10, 50)
    assert res.rank == 1 and res.achieved_relative_error <= 1e-10

    t = _planted(orc, (5, 5, 5), (2, 2, 2), 110, 1e-6)
    res = vie.tucker_cp(dft, t, (5, 5, 5), (1, 1, 1), 1e-4, 400)
    assert res.hosvd_relative_error > 0
    assert res.achieved_relative_error <= 10 * res.hosvd_relative_error

    t = _planted(orc, (6, 6, 6), (3, 3, 3), 120, 1e-4)
    res = vie.tucker_cp(dft, t, (6, 6, 6), (1, 1, 1), 1e-2, 200)
    h = res.hosvd_relative_error
    combined = np.hypot(h, res.core_cp_relative_error * np.sqrt(max(0.0, 1 - h * h)))
    assert abs(res.achieved_relative_error - combined) <= 1e-10
    assert res.achieved_relative_error >= h - 1e-13

    t = _planted(orc, (5, 4, 6), (2, 2, 2), 130, 1e-5)
    res = vie.tucker_cp(dft, t, (5, 4, 6), (1, 1, 1), 1e-3, 200)
    err = np.linalg.norm(_cp_reconstruct(res.factors) - t) / np.linalg.norm(t)
    assert abs(err - res.achieved_relative_error) <= 1e-12


@pytest.mark.parametrize("dims,ranks,seed,noise,tol,iters", [
    ((9, 8, 10), (3, 2, 4), 500, 1e-5, 1e-3, 200),
    ((12, 10, 8), (4, 4, 3), 510, 1e-7, 1e-5, 300),
    ((10, 9, 8), (3, 3, 3), 530, 1e-6, 1e-4, 150),
])
def test_tucker_cp_matches_oracle(vie, dft, orc, dims, ranks, seed, noise, tol, iters):
    """CP rank <= every core rank: the initial factors are all singular vectors, so the CP-ALS
    trajectory is independent of the HOSVD's column phases and the sweeps agree with the
    oracle's to rounding.  With stall_tol = 0 the last sweeps are decided by rounding noise
    (the run stops at the first non-decrease), so the traces are compared over their common
    prefix and the final errors directly."""
    t = _planted(orc, dims, ranks, seed, noise)
    o = orc.tucker_cp(t, dims, tol, iters, 1)
    for src in ("host", "device"):
        tt = t
        if src == "device":
            import torch

            tt = torch.from_numpy(t).cuda()
        a = vie.tucker_cp(dft, tt, dims, (1, 1, 1), tol, iters, 1)
        assert a.rank == o.rank
        n = min(len(a.cp_error_trace), len(o.trace))
        assert n >= 1 and np.max(np.abs(a.cp_error_trace[:n] - o.trace[:n])) <= 1e-8
        for x, y in [(a.hosvd_relative_error, o.hosvd_relative_error),
                     (a.core_cp_relative_error, o.core_cp_relative_error),
                     (a.achieved_relative_error, o.achieved_relative_error)]:
            assert abs(x - y) <= 1e-8 * max(1.0, y) + 1e-12
        ra, ro = _cp_reconstruct(a.factors), _cp_reconstruct(o.factors)
        assert np.linalg.norm(ra - ro) <= 1e-6 * np.linalg.norm(t)


def test_tucker_cp_padded_rank(vie, dft, orc):
    """CP rank above the core ranks: the extra initial columns are seeded Gaussians expressed in
    the HOSVD basis, whose column phases are a convention of the SVD (the reference's Eigen, the
    oracle's QR + Jacobi, the device Gram + Jacobi differ), so the fits are different valid
    ones: same rank, both converge, the error decomposition holds (test_decomp.cpp:247-258)."""
    dims = (8, 8, 8)
    t = _planted(orc, dims, (3, 3, 3), 520, 1e-6)
    o = orc.tucker_cp(t, dims, 1e-4, 100, 1, 5)
    a = vie.tucker_cp(dft, t, dims, (1, 1, 1), 1e-4, 100, 1, 5)
    assert a.rank == o.rank == 5
    assert abs(a.hosvd_relative_error - o.hosvd_relative_error) <= 1e-10
    assert a.core_cp_relative_error <= 1e-4 and o.core_cp_relative_error <= 1e-4
    h = a.hosvd_relative_error
    combined = np.hypot(h, a.core_cp_relative_error * np.sqrt(max(0.0, 1 - h * h)))
    assert abs(a.achieved_relative_error - combined) <= 1e-10


def test_tucker_cp_operator_matches_oracle_fit(vie, dft, orc):
    """build_operator_spectra with opts.tucker_cp (operator.hpp:165-168): every component fitted
    by tucker_cp on the device; the matvec equals the oracle's on the oracle's own fits."""
    dims = (6, 5, 4)
    fam = make_family(N, PWC, dims, 90)
    comps, par, _ = vie.component_table(N, PWC)
    tol, iters = 1e-6, 200
    forms, oforms = [], []
    for c in range(len(comps)):
        res = vie.tucker_cp(dft, fam[c], dims, par[c], tol, iters)
        forms.append(res.form)
        o = orc.tucker_cp(fam[c], dims, tol, iters)
        R = o.rank
        core = np.zeros((R, R, R), np.complex128)
        core[np.arange(R), np.arange(R), np.arange(R)] = 1.0
        wf = [orc.transform_factor(o.factors[q], par[c][q]) for q in range(3)]
        oforms.append(orc.Form(core, *wf))
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    x = random_field(PWC, dims, 31)
    import torch

    y = vie.apply_operator(op, torch.from_numpy(x).cuda()).cpu().numpy()
    y_ref = orc.apply_operator_tucker(N, PWC, dims, oforms, x)
    assert rel(y_ref, y) <= 1e-8
