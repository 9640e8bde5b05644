"""GPU parity of Tucker+CP components (vie_tucker_from_cp): the fused matvec on
CP forms against the oracle on the same forms (decompress_cp == Tucker with the
superdiagonal core, pinned in test_oracle_cp.py).  Bar: relative l2 <= 1e-10."""
import numpy as np
import pytest

from tests.helpers import rel

pytestmark = pytest.mark.gpu

N, K, PWC, PWL = 0, 1, 0, 1


@pytest.fixture(scope="module")
def vie():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as v

    return v


@pytest.mark.parametrize("kind,basis,dims,R", [(N, PWC, (5, 4, 6), 4), (K, PWC, (4, 6, 5), 3),
                                               (N, PWL, (4, 3, 5), 3)])
def test_cp_matvec_matches_oracle(vie, orc, kind, basis, dims, R):
    import torch

    dft = vie.DftService(0)
    comps, par, _ = vie.component_table(kind, basis)
    rng = np.random.default_rng(17)
    forms, oforms = [], []
    diag = np.zeros((R, R, R), np.complex128)
    diag[np.arange(R), np.arange(R), np.arange(R)] = 1.0
    for c in range(len(comps)):
        ws = [rng.standard_normal((dims[q], R)) + 1j * rng.standard_normal((dims[q], R)) for q in range(3)]
        for q in range(3):
            if par[c][q] < 0:
                ws[q][0, :] = 0.0  # odd-parity rows (components.hpp:51-65)
        forms.append(vie.tucker_cp_form(dft, dims, ws, par[c]))
        wh = [orc.transform_factor(ws[q], int(par[c][q])) for q in range(3)]
        oforms.append(orc.Form(diag, *wh))
    op = vie.build_operator_spectra(kind, basis, dims, comps, forms, dft)
    S = vie.ncur(basis)
    nv = int(np.prod(dims))
    x = rng.standard_normal(S * nv) + 1j * rng.standard_normal(S * nv)
    y = vie.apply_operator(op, torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
    assert rel(y.cpu().numpy(), ref) <= 1e-10


def test_cp_form_errors(vie):
    dft = vie.DftService(0)
    w = np.ones((3, 2), np.complex128)
    with pytest.raises(ValueError):
        vie.tucker_cp_form(dft, (3, 3, 3), [w, w, np.ones((3, 3))], (1, 1, 1))
    with pytest.raises(ValueError):
        vie.tucker_cp_form(dft, (3, 3, 3), [w, w, w], (1, -1, 1))  # odd axis with a nonzero row 0
