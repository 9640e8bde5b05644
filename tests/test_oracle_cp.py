"""Pins the oracle's decompress_cp (operator.hpp:248-261, the Tucker+CP spectrum)
against the CP definition (cp_reconstruct, decomp.hpp:143-148) and against the
Tucker decompressor with the superdiagonal core -- the identity the device path
relies on (vie_tucker_from_cp).  No GPU."""
import numpy as np


def rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_decompress_cp_matches_definition_and_superdiagonal_tucker(orc):
    rng = np.random.default_rng(8)
    edims, R = (6, 4, 10), 5
    ws = [rand_c(rng, m, R) for m in edims]
    s = orc.decompress_cp(edims, ws)
    ref = np.einsum("il,jl,kl->ijk", *ws).reshape(-1, order="F")
    assert np.linalg.norm(s - ref) <= 1e-13 * np.linalg.norm(ref)
    core = np.zeros((R, R, R), np.complex128)
    core[np.arange(R), np.arange(R), np.arange(R)] = 1.0
    t = orc.decompress_tucker(edims, orc.Form(core, *ws))
    assert np.linalg.norm(s - t) <= 1e-13 * np.linalg.norm(ref)


def test_decompress_cp_rank_zero_is_zero(orc):  # operator.hpp:252-255
    edims = (2, 2, 2)
    ws = [np.zeros((2, 0), np.complex128)] * 3
    assert np.all(orc.decompress_cp(edims, ws) == 0)


# ---- cp_als / tucker_cp (decomp.hpp:237-373), the reference's tests restated
# (test_decomp.cpp:174-267).  random_orthonormal = thin Q of random_matrix (test_util.hpp:27-31).
def _cp_reconstruct(fs):
    return np.einsum("il,jl,kl->ijk", *fs).reshape(-1, order="F")


def _outer3(orc, dims, seeds):
    return _cp_reconstruct([orc.random_matrix(dims[q], 1, seeds[q]) for q in range(3)])


def _ortho(orc, rows, cols, seed):
    return np.linalg.qr(orc.random_matrix(rows, cols, seed))[0]


def _planted(orc, dims, ranks, seed, noise):  # test_decomp.cpp:16-27
    core = orc.random_tensor(*ranks, seed).reshape(ranks, order="F")
    us = [_ortho(orc, dims[q], ranks[q], seed + 1 + q) for q in range(3)]
    t = np.einsum("abg,ia,jb,kg->ijk", core, *us).reshape(-1, order="F")
    if noise > 0:
        n = orc.random_tensor(*dims, seed + 4)
        t = t + noise * np.linalg.norm(t) / np.linalg.norm(n) * n
    return t


def test_cp_als_exact_rank_one(orc):  # test_decomp.cpp:174-179
    t = _outer3(orc, (5, 4, 6), (70, 71, 72))
    res = orc.cp_als(t, (5, 4, 6), 1, 10)
    assert res.trace[-1] <= 1e-10


def test_cp_als_exact_rank_two_well_separated(orc):  # test_decomp.cpp:181-189
    v = [_ortho(orc, 6, 2, 80 + q) for q in range(3)]
    v[2][:, 0] *= 3.0
    t = _cp_reconstruct(v)
    res = orc.cp_als(t, (6, 6, 6), 2, 200, 1e-15)
    assert res.trace[-1] <= 1e-8


def test_cp_als_rank_deficit_bounded_below_and_monotone(orc):  # test_decomp.cpp:191-213
    v = [_ortho(orc, 2, 2, 90 + q) for q in range(3)]
    v[2][:, 0] *= 2.0
    t = _cp_reconstruct(v)
    tn = np.linalg.norm(t)
    T = t.reshape((2, 2, 2), order="F")
    lower = 0.0
    for mode in range(3):
        s = np.linalg.svd(np.moveaxis(T, mode, 0).reshape(2, -1), compute_uv=False)
        lower = max(lower, np.sqrt(np.sum(s[1:] ** 2)) / tn)
    assert lower > 0
    res = orc.cp_als(t, (2, 2, 2), 1, 50, 1e-15)
    assert res.trace[-1] >= lower * (1 - 1e-10)
    assert np.all(np.diff(res.trace) <= 1e-12)


def test_cp_als_monotone_on_random_tensor(orc):  # test_decomp.cpp:215-220
    res = orc.cp_als(orc.random_tensor(5, 5, 5, 95), (5, 5, 5), 3, 60, 1e-15)
    assert np.all(np.diff(res.trace) <= 1e-12)


def test_cp_als_ill_posed_rank_flagged(orc):  # test_decomp.cpp:222-228
    res = orc.cp_als(orc.random_tensor(3, 3, 3, 96), (3, 3, 3), 10, 3)
    assert res.ill_posed
    assert res.factors[0].shape[1] == 10
    assert np.all(np.isfinite(res.trace))


def test_cp_als_definition(orc):
    """The returned factors reproduce the last trace entry (cp_reconstruct of the factors)."""
    t = orc.random_tensor(4, 5, 3, 11)
    res = orc.cp_als(t, (4, 5, 3), 4, 25, 0.0)
    err = np.linalg.norm(_cp_reconstruct(res.factors) - t) / np.linalg.norm(t)
    assert abs(err - res.trace[-1]) <= 1e-12


def test_tucker_cp_rank_one_tensor(orc):  # test_decomp.cpp:230-236
    t = _outer3(orc, (5, 5, 5), (100, 101, 102))
    res = orc.tucker_cp(t, (5, 5, 5), 1e-10, 50)
    assert res.rank == 1
    assert res.achieved_relative_error <= 1e-10


def test_tucker_cp_near_hosvd_error_on_noisy_low_rank(orc):  # test_decomp.cpp:238-245
    t = _planted(orc, (5, 5, 5), (2, 2, 2), 110, 1e-6)
    res = orc.tucker_cp(t, (5, 5, 5), 1e-4, 400)
    assert res.hosvd_relative_error > 0
    assert res.achieved_relative_error <= 10 * res.hosvd_relative_error


def test_tucker_cp_error_decomposition(orc):  # test_decomp.cpp:247-258
    t = _planted(orc, (6, 6, 6), (3, 3, 3), 120, 1e-4)
    res = orc.tucker_cp(t, (6, 6, 6), 1e-2, 200)
    h = res.hosvd_relative_error
    combined = np.hypot(h, res.core_cp_relative_error * np.sqrt(max(0.0, 1 - h * h)))
    assert abs(res.achieved_relative_error - combined) <= 1e-10
    assert res.achieved_relative_error >= h - 1e-13


def test_tucker_cp_reconstruct_matches_cp_of_merged_factors(orc):  # test_decomp.cpp:260-267
    t = _planted(orc, (5, 4, 6), (2, 2, 2), 130, 1e-5)
    res = orc.tucker_cp(t, (5, 4, 6), 1e-3, 200)
    a = _cp_reconstruct(res.factors)
    assert a.shape == t.shape
    err = np.linalg.norm(a - t) / np.linalg.norm(t)
    assert abs(err - res.achieved_relative_error) <= 1e-12
