"""The library's cp_als (cp_als.cu, the CP fitting of tucker_cp: host code on the HOSVD core,
decomp.hpp:237-298) against the oracle restatement and the reference's CpAls tests
(test_decomp.cpp:174-228).  Host logic only: runs without a GPU."""
import numpy as np
import pytest

from tests.test_oracle_cp import _cp_reconstruct, _ortho, _outer3


@pytest.fixture(scope="module")
def vie():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as v

    return v


@pytest.mark.parametrize("dims,r,iters,stall,seed", [((5, 5, 5), 3, 60, 1e-15, 95), ((4, 6, 5), 2, 40, 0.0, 7),
                                                     ((4, 6, 5), 8, 40, 0.0, 7), ((6, 3, 4), 5, 80, 1e-12, 3),
                                                     ((3, 3, 3), 10, 3, 1e-12, 96), ((7, 2, 5), 1, 30, 0.0, 4)])
def test_cp_als_matches_oracle(vie, orc, dims, r, iters, stall, seed):
    t = orc.random_tensor(*dims, seed)
    a = vie.cp_als(t, dims, r, iters, stall)
    o = orc.cp_als(t, dims, r, iters, stall)
    assert a.ill_posed_rank == o.ill_posed and a.converged == o.converged
    assert len(a.rel_error_trace) == len(o.trace)
    assert np.max(np.abs(a.rel_error_trace - o.trace)) <= 1e-10
    # same decomposition: the reconstructions agree (column phases are free)
    ra, ro = _cp_reconstruct(a.factors), _cp_reconstruct(o.factors)
    assert np.linalg.norm(ra - ro) <= 1e-8 * np.linalg.norm(t)


def test_cp_als_reference_cases(vie, orc):  # test_decomp.cpp:174-228 through the library
    t = _outer3(orc, (5, 4, 6), (70, 71, 72))
    assert vie.cp_als(t, (5, 4, 6), 1, 10).rel_error_trace[-1] <= 1e-10
    v = [_ortho(orc, 6, 2, 80 + q) for q in range(3)]
    v[2][:, 0] *= 3.0
    assert vie.cp_als(_cp_reconstruct(v), (6, 6, 6), 2, 200, 1e-15).rel_error_trace[-1] <= 1e-8
    res = vie.cp_als(orc.random_tensor(5, 5, 5, 95), (5, 5, 5), 3, 60, 1e-15)
    assert np.all(np.diff(res.rel_error_trace) <= 1e-12)
    ill = vie.cp_als(orc.random_tensor(3, 3, 3, 96), (3, 3, 3), 10, 3)
    assert ill.ill_posed_rank and ill.factors[0].shape == (3, 10)


def test_cp_als_edge_cases(vie):
    z = vie.cp_als(np.zeros(8, complex), (2, 2, 2), 2, 5)
    assert z.converged and list(z.rel_error_trace) == [0.0] and np.all(z.factors[0] == 0)
    r0 = vie.cp_als(np.ones(8, complex), (2, 2, 2), 0, 5)
    assert not r0.converged and list(r0.rel_error_trace) == [1.0]
    with pytest.raises(ValueError):
        vie.cp_als(np.ones(8, complex), (2, 2, 2), -1, 5)
    with pytest.raises(ValueError):
        vie.cp_als(np.ones(8, complex), (2, 2, 2), 1, 0)
