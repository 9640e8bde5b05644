"""tucker_compress on the device (vie_tucker_compress) against the oracle's
hosvd (decomp.hpp:160-176) and the reference's compression tests
(test_decomp.cpp, test_fft_operator.cpp:192-209)."""
import numpy as np
import pytest

from tests.helpers import flat, make_family, random_field, rel, tucker_reconstruct

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


def planted(orc, dims, ranks, seed, noise):  # test_decomp.cpp:16-27
    core = orc.random_tensor(*ranks, seed)
    us = [np.linalg.qr(orc.random_matrix(dims[q], ranks[q], seed + 1 + q))[0] for q in range(3)]
    t = tucker_reconstruct(core, ranks, *us)
    if noise:
        nz = orc.random_tensor(*dims, seed + 4)
        t = t + noise * np.linalg.norm(t) / np.linalg.norm(nz) * nz
    return t


@pytest.mark.parametrize("rule", [0, 1])
def test_ranks_match_oracle_hosvd(vie, dft, orc, rule):
    for trial in range(4):
        dims = (9, 8, 10)
        t = planted(orc, dims, (3, 2, 4), 1000 + 7 * trial, 1e-5)
        for tol in (1e-2, 1e-4):
            core, us = orc.hosvd(t, dims, tol, rule)
            f = vie.tucker_compress(dft, t, dims, (1, 1, 1), tol, rule)
            assert list(f.ranks) == [u.shape[1] for u in us], (trial, tol)


def test_compressed_operator_error_tracks_tolerance(vie, dft, orc):  # test_fft_operator.cpp:192-209
    dims = (4, 4, 4)
    fam = make_family(N, PWC, dims, 70)
    comps, par, _ = vie.component_table(N, PWC)
    tol = 1e-4
    forms = [vie.tucker_compress(dft, fam[c], dims, par[c], tol) for c in range(6)]
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(6)]
    x = random_field(PWC, dims, 71)
    ref = orc.apply_operator_dense(N, PWC, dims, spectra, x)
    assert rel(ref, vie.apply_operator(op, x)) < 10 * tol


def test_compress_tight_tolerance_matches_dense(vie, dft, orc):  # test_fft_operator.cpp:172-190
    dims = (3, 3, 4)
    fam = make_family(N, PWC, dims, 60)
    comps, par, _ = vie.component_table(N, PWC)
    forms = [vie.tucker_compress(dft, fam[c], dims, par[c], 1e-10) for c in range(6)]
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(6)]
    x = random_field(PWC, dims, 61)
    assert rel(orc.apply_operator_dense(N, PWC, dims, spectra, x), vie.apply_operator(op, x)) < 1e-8


def test_compress_errors(vie, dft):
    with pytest.raises(ValueError):
        vie.tucker_compress(dft, np.zeros(0, complex), (0, 2, 2), (1, 1, 1))
    with pytest.raises(ValueError):
        vie.tucker_compress(dft, np.ones(8, complex), (2, 2, 2), (1, 1, 1), -1.0)
