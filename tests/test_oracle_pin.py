"""Pins the CPU oracle against the reference's own known-answer tests and an
independent numpy/scipy path (no GPU).  Each test cites the reference test it
restates (paths relative to /root/reference/proj/tests)."""
import numpy as np
import pytest

from tests.helpers import (flat, make_family, make_component_tensor, np_apply_dense, np_circulant_embed,
                           np_fft3, random_field, rel, tucker_reconstruct, unflat)

N, K, PWC, PWL = 0, 1, 0, 1


# ---------------------------------------------------------------- embedding
def test_embed_smallest_case_enumerated(orc):  # test_fft_operator.cpp:50-63
    e = orc.circulant_embed(np.array([2 + 1j]), (1, 1, 1), (1, 1, 1))
    assert e.size == 8 and e[0] == 2 + 1j and np.all(e[1:] == 0)


def test_embed_1d_toeplitz_column(orc):  # test_fft_operator.cpp:65-75
    t = np.array([1.0, 0.5 - 0.25j])
    e = unflat(orc.circulant_embed(t, (2, 1, 1), (1, 1, 1)), (4, 2, 2))
    assert e[0, 0, 0] == t[0] and e[1, 0, 0] == t[1] and e[2, 0, 0] == 0 and e[3, 0, 0] == t[1]


def test_embed_odd_parity_flips_sign(orc):  # test_fft_operator.cpp:77-87
    t = np.array([0.0, 2.0, 3.0])
    e = unflat(orc.circulant_embed(t, (3, 1, 1), (-1, 1, 1)), (6, 2, 2))
    assert e[4, 0, 0] == -3.0 and e[5, 0, 0] == -2.0


def test_embed_matches_numpy(orc):
    rng = np.random.default_rng(3)
    dims = (3, 4, 5)
    t = rng.standard_normal(60) + 1j * rng.standard_normal(60)
    for sign in [(1, 1, 1), (-1, 1, -1), (1, -1, 1)]:
        assert np.array_equal(orc.circulant_embed(t, dims, sign), np_circulant_embed(t, dims, sign))


# ---------------------------------------------------------------- DFT service
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 17, 25, 30, 31, 64, 100, 186, 238, 250, 400, 480])
def test_fft1_matches_numpy(orc, n):  # fft.hpp:32-40 conventions
    rng = np.random.default_rng(n)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert rel(np.fft.fft(v), orc.fft1(v)) < 1e-13
    assert rel(np.fft.ifft(v), orc.fft1(v, inverse=True)) < 1e-13


def test_fft3_matches_numpy_and_roundtrips(orc):
    rng = np.random.default_rng(1)
    dims = (6, 10, 8)
    v = rng.standard_normal(480) + 1j * rng.standard_normal(480)
    f = orc.fft3(v, dims)
    assert rel(np_fft3(v, dims), f) < 1e-13
    assert rel(v, orc.fft3(f, dims, inverse=True)) < 1e-14


# ---------------------------------------------------------------- tables
def test_pwc_tables_match_reference(orc):  # components.hpp:46-92, operator.hpp:205-219
    comps, par, blocks = orc.component_table(N, PWC)
    assert [tuple(c[:2]) for c in comps] == [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    assert [tuple(p) for p in par] == [(1, 1, 1), (-1, -1, 1), (-1, 1, -1), (1, 1, 1), (1, -1, -1), (1, 1, 1)]
    # FFT coefficient = dense_sign * sigma; reference: N -> (a,a,s) / (a,b,s),(b,a,s)
    coeffs = [(t, s, c, ds * int(np.prod(par[c]))) for t, s, c, ds in blocks]
    assert coeffs == [(0, 0, 0, 1), (0, 1, 1, 1), (1, 0, 1, 1), (0, 2, 2, 1), (2, 0, 2, 1), (1, 1, 3, 1),
                      (1, 2, 4, 1), (2, 1, 4, 1), (2, 2, 5, 1)]
    comps, par, blocks = orc.component_table(K, PWC)
    assert [tuple(c[:2]) for c in comps] == [(0, 1), (0, 2), (1, 2)]
    assert [tuple(p) for p in par] == [(1, 1, -1), (1, -1, 1), (-1, 1, 1)]
    coeffs = [(t, s, c, ds * int(np.prod(par[c]))) for t, s, c, ds in blocks]
    # reference K: (a,b,sigma), (b,a,-sigma), sigma = -1
    assert coeffs == [(0, 1, 0, -1), (1, 0, 0, 1), (0, 2, 1, -1), (2, 0, 1, 1), (1, 2, 2, -1), (2, 1, 2, 1)]


def test_pwl_table_counts(orc):  # PAPER.md:127 (60 unique N, 30 unique K, 144 blocks)
    comps, par, blocks = orc.component_table(N, PWL)
    assert len(comps) == 60 and len(blocks) == 144
    assert len({(t, s) for t, s, _, _ in blocks}) == 144
    comps, par, blocks = orc.component_table(K, PWL)
    assert len(comps) == 30 and len(blocks) == 96  # K_qq = 0: 6 x 16 diagonal blocks absent


# ---------------------------------------------------------------- operator
def test_transform_factors_matches_dense_path(orc):  # test_fft_operator.cpp:89-102
    comps, par, _ = orc.component_table(N, PWC)
    p = par[1]  # N xy
    t = make_component_tensor(p, (4, 4, 4), 7)
    core, us = orc.hosvd(t, (4, 4, 4), 0.0)
    uh = [orc.transform_factor(us[q], int(p[q])) for q in range(3)]
    via = tucker_reconstruct(core, [u.shape[1] for u in us], *uh)
    dense = orc.dense_spectrum(t, (4, 4, 4), p)
    assert rel(dense, via) < 1e-12


def test_transform_factor_octant_symmetry(orc):
    # U^(m-p) = sign * U^(p) when row 0 vanishes on odd axes
    u = orc.random_matrix(9, 3, 5)
    for sign in (1, -1):
        uu = u.copy()
        if sign < 0:
            uu[0] = 0
        h = orc.transform_factor(uu, sign)
        m = 18
        for p in range(1, 18):
            assert np.allclose(h[m - p], sign * h[p], atol=1e-13)
        if sign < 0:
            assert np.allclose(h[0], 0, atol=1e-13) and np.allclose(h[9], 0, atol=1e-13)


@pytest.mark.parametrize("kind", [N, K])
@pytest.mark.parametrize("basis", [PWC, PWL])
def test_dense_matches_bttb(orc, kind, basis):  # test_fft_operator.cpp:132-149
    dims = (3, 3, 4) if basis == PWC else (2, 3, 2)
    fam = make_family(kind, basis, dims, 30)
    a = orc.dense_bttb(kind, basis, dims, fam)
    spectra = [orc.dense_spectrum(fam[c], dims, orc.component_table(kind, basis)[1][c]) for c in range(len(fam))]
    for trial in range(3):
        x = random_field(basis, dims, 40 + 3 * trial)
        y = orc.apply_operator_dense(kind, basis, dims, spectra, x)
        assert rel(a @ x, y) < 1e-12
        assert rel(np_apply_dense(kind, basis, dims, fam, x), y) < 1e-12


def test_diagonalization_identity_small_grids(orc):  # test_fft_operator.cpp:153-170
    seed = 50
    _, par, _ = orc.component_table(N, PWC)
    for n1 in range(1, 5):
        for n2 in (1, 4):
            for n3 in (2, 4):
                seed += 17
                dims = (n1, n2, n3)
                fam = make_family(N, PWC, dims, seed)
                a = orc.dense_bttb(N, PWC, dims, fam)
                spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(6)]
                x = random_field(PWC, dims, seed + 1)
                y = orc.apply_operator_dense(N, PWC, dims, spectra, x)
                assert rel(a @ x, y) < 1e-12, dims


@pytest.mark.parametrize("basis", [PWC, PWL])
def test_hosvd_decompress_agrees_with_dense(orc, basis):  # test_fft_operator.cpp:172-190
    dims = (3, 3, 4) if basis == PWC else (2, 3, 2)
    fam = make_family(N, basis, dims, 60)
    _, par, _ = orc.component_table(N, basis)
    forms = []
    for c, t in enumerate(fam):
        core, us = orc.hosvd(t, dims, 1e-10)
        uh = [orc.transform_factor(us[q], int(par[c][q])) for q in range(3)]
        forms.append(orc.Form(core, *uh))
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(len(fam))]
    x = random_field(basis, dims, 61)
    ref = orc.apply_operator_dense(N, basis, dims, spectra, x)
    y = orc.apply_operator_tucker(N, basis, dims, forms, x)
    assert rel(ref, y) < 1e-8


def test_error_tracks_compression_tolerance(orc):  # test_fft_operator.cpp:192-209
    dims = (4, 4, 4)
    fam = make_family(N, PWC, dims, 70)
    _, par, _ = orc.component_table(N, PWC)
    forms = []
    for c, t in enumerate(fam):
        core, us = orc.hosvd(t, dims, 1e-4)
        forms.append(orc.Form(core, *[orc.transform_factor(us[q], int(par[c][q])) for q in range(3)]))
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(6)]
    x = random_field(PWC, dims, 71)
    assert rel(orc.apply_operator_dense(N, PWC, dims, spectra, x),
               orc.apply_operator_tucker(N, PWC, dims, forms, x)) < 10 * 1e-4


def test_linearity(orc):  # test_fft_operator.cpp:211-234
    dims = (3, 2, 3)
    fam = make_family(N, PWC, dims, 80)
    _, par, _ = orc.component_table(N, PWC)
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(6)]
    x = random_field(PWC, dims, 81)
    y = random_field(PWC, dims, 82)
    lam = 0.7 - 1.3j
    A = lambda v: orc.apply_operator_dense(N, PWC, dims, spectra, v)
    assert rel(A(x) + lam * A(y), A(x + lam * y)) < 1e-12


@pytest.mark.parametrize("kind", [N, K])
def test_adjoint_consistency(orc, kind):  # test_fft_operator.cpp:238-263
    dims = (3, 2, 4)
    fam = make_family(kind, PWC, dims, 90)
    _, par, _ = orc.component_table(kind, PWC)
    a = orc.dense_bttb(kind, PWC, dims, fam)
    ah = orc.dense_bttb(kind, PWC, dims, [np.conj(t) for t in fam])
    assert np.linalg.norm(a.conj().T - ah) / np.linalg.norm(a) < 1e-13
    spectra = [orc.dense_spectrum(fam[c], dims, par[c]) for c in range(len(fam))]
    x = random_field(PWC, dims, 91)
    y = random_field(PWC, dims, 92)
    ax = orc.apply_operator_dense(kind, PWC, dims, spectra, x)
    lhs = np.vdot(ax, y)
    rhs = np.vdot(x, a.conj().T @ y)
    assert abs(lhs - rhs) / abs(lhs) < 1e-10


def test_pwl_n_operator_is_symmetric(orc):
    # reciprocity: the PWL N Galerkin matrix is complex-symmetric (A^T = A) for
    # physical (even-kernel) tensors built with per-block parity; our table's
    # dense signs encode exactly this.
    dims = (2, 2, 3)
    fam = make_family(N, PWL, dims, 11)
    a = orc.dense_bttb(N, PWL, dims, fam)
    # the family is random, so only the block sign/parity structure is exercised:
    # blocks (t,s) and (s,t) come from the same stored component.
    _, _, blocks = orc.component_table(N, PWL)
    comp_of = {(t, s): c for t, s, c, _ in blocks}
    for (t, s), c in comp_of.items():
        assert comp_of[(s, t)] == c
    assert np.isfinite(a).all()


# ---------------------------------------------------------------- system
@pytest.mark.parametrize("basis", [PWC, PWL])
def test_apply_system_matches_dense_system(orc, basis):  # test_solver.cpp:153-180
    dims = (3, 3, 4) if basis == PWC else (2, 2, 3)
    fam = make_family(N, basis, dims, 5)
    _, par, _ = orc.component_table(N, basis)
    forms = []
    for c, t in enumerate(fam):
        core, us = orc.hosvd(t, dims, 0.0)
        forms.append(orc.Form(core, *[orc.transform_factor(us[q], int(par[c][q])) for q in range(3)]))
    nv = int(np.prod(dims))
    S = orc.ncur(basis)
    rng = np.random.default_rng(4)
    eps = 1 + rng.uniform(0, 5, nv) - 1j * rng.uniform(0, 1, nv)
    inv_v = 0.37
    bttb = orc.dense_bttb(N, basis, dims, fam) * inv_v
    g = np.array([1.0 if (basis == PWC or q % 4 == 0) else 1 / 12 for q in range(S)])
    epsv = np.concatenate([eps * g[q] for q in range(S)])
    chiv = np.concatenate([eps - 1 for _ in range(S)])
    A = np.diag(epsv) - np.diag(chiv) @ bttb
    x = random_field(basis, dims, 20)
    y = orc.apply_system_tucker(basis, dims, forms, eps, inv_v, x)
    assert rel(A @ x, y) < 1e-12


def test_apply_system_zero_contrast_identity(orc):  # test_solver.cpp:141-151
    dims = (3, 3, 3)
    fam = make_family(N, PWC, dims, 9)
    _, par, _ = orc.component_table(N, PWC)
    forms = []
    for c, t in enumerate(fam):
        core, us = orc.hosvd(t, dims, 0.0)
        forms.append(orc.Form(core, *[orc.transform_factor(us[q], int(par[c][q])) for q in range(3)]))
    x = random_field(PWC, dims, 10)
    y = orc.apply_system_tucker(PWC, dims, forms, np.ones(27, complex), 100.0, x)
    assert rel(x, y) < 1e-13


# ---------------------------------------------------------------- GMRES
def test_gmres_identity_one_iteration(orc):  # test_solver.cpp:31-38
    rhs = orc.random_matrix(20, 1, 1)[:, 0]
    r = orc.gmres(lambda v: v, rhs)
    assert r.converged and r.iterations == 1 and rel(rhs, r.solution) < 1e-12


def test_gmres_diagonal(orc):  # test_solver.cpp:40-53
    d = np.array([complex(i + 1.0, 0.5 * i) for i in range(10)])
    rhs = orc.random_matrix(10, 1, 2)[:, 0]
    r = orc.gmres(lambda v: d * v, rhs, tol=1e-12)
    assert r.converged and rel(rhs / d, r.solution) < 1e-10


def test_gmres_restarts(orc):  # test_solver.cpp:55-68
    a = orc.random_matrix(30, 30, 3)
    a = a @ a.conj().T / 30 + 4 * np.eye(30)
    rhs = orc.random_matrix(30, 1, 4)[:, 0]
    r = orc.gmres(lambda v: a @ v, rhs, tol=1e-9, inner=5, outer=100)
    assert r.converged and np.linalg.norm(a @ r.solution - rhs) / np.linalg.norm(rhs) <= 2e-9


def test_gmres_history_monotone(orc):  # test_solver.cpp:70-82
    a = orc.random_matrix(25, 25, 5) + 6 * np.eye(25)
    rhs = orc.random_matrix(25, 1, 6)[:, 0]
    r = orc.gmres(lambda v: a @ v, rhs, tol=1e-14, inner=25, outer=1)
    h = r.residual_history
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))


def test_gmres_reported_residual(orc):  # test_solver.cpp:84-97
    a = orc.random_matrix(20, 20, 7) + 5 * np.eye(20)
    rhs = orc.random_matrix(20, 1, 8)[:, 0]
    r = orc.gmres(lambda v: a @ v, rhs, tol=1e-8)
    assert r.converged
    ext = np.linalg.norm(a @ r.solution - rhs) / np.linalg.norm(rhs)
    assert abs(ext - r.final_relative_residual) <= 1e-10 * max(1, ext)
    assert abs(r.residual_history[-1] - ext) <= 1e-10


def test_gmres_nonconvergence_flag(orc):  # test_solver.cpp:99-114
    a = np.zeros((40, 40), complex)
    for i in range(39):
        a[i + 1, i] = 1
    a[0, 39] = 1
    rhs = np.zeros(40, complex)
    rhs[0] = 1
    r = orc.gmres(lambda v: a @ v, rhs, tol=1e-12, inner=3, outer=2)
    assert not r.converged and r.solution.size == 40


def test_gmres_warm_start_and_precond(orc):  # test_scene_io.cpp:107-139
    d = np.array([complex(2 + i, 0.3) for i in range(8)])
    rhs = orc.random_matrix(8, 1, 1)[:, 0]
    cold = orc.gmres(lambda v: d * v, rhs, tol=1e-10)
    warm = orc.gmres(lambda v: d * v, rhs, tol=1e-10, x0=cold.solution)
    assert cold.converged and warm.converged and warm.iterations == 0
    d2 = np.array([complex(1 + 3 * i, -0.5 * i) for i in range(12)])
    rhs2 = orc.random_matrix(12, 1, 2)[:, 0]
    r = orc.gmres(lambda v: d2 * v, rhs2, tol=1e-12, precond=lambda v: v / d2)
    assert r.converged and r.iterations == 1
    assert np.linalg.norm(d2 * r.solution - rhs2) / np.linalg.norm(rhs2) < 1e-12


def test_gmres_errors(orc):  # solver.hpp:37-39
    with pytest.raises(orc.OracleError):
        orc.gmres(lambda v: v, np.array([np.nan, 1.0]))
    with pytest.raises(orc.OracleError):
        orc.gmres(lambda v: v, np.ones(3), inner=0)
    r = orc.gmres(lambda v: v, np.zeros(4))
    assert r.converged and np.all(r.solution == 0)


# ---------------------------------------------------------------- HOSVD
def test_svd_values_match_numpy(orc):  # test_decomp.cpp:64-73 (wide path)
    for shape, seed in [((4, 40), 3), ((40, 4), 4), ((7, 9), 5)]:
        m = orc.random_matrix(shape[0], shape[1], seed)
        rank, s = orc.truncated_svd_values(m, 0.0)
        assert rank == min(shape)
        assert np.allclose(s, np.linalg.svd(m, compute_uv=False), rtol=1e-12, atol=1e-12)


def test_truncation_rules(orc):  # test_decomp.cpp:31-62
    u = orc.random_matrix(6, 1, 1)
    v = orc.random_matrix(5, 1, 2)
    for tol in (1e-1, 1e-6, 0.5):
        assert orc.truncated_svd_values(u @ v.T, tol)[0] == 1
    assert orc.truncated_svd_values(np.eye(4), 0.0, rule=0)[0] == 4
    assert orc.truncated_svd_values(np.eye(4), 0.0, rule=1)[0] == 4
    assert orc.truncated_svd_values(np.diag([1.0, 1e-3, 1e-9]), 1e-6, rule=0)[0] == 2
    with pytest.raises(orc.OracleError):
        orc.truncated_svd_values(np.eye(2), -1.0)


def test_hosvd_known_answers(orc):  # test_decomp.cpp:75-110
    t = np.einsum("i,j,k->ijk", orc.random_matrix(5, 1, 4)[:, 0], orc.random_matrix(6, 1, 5)[:, 0],
                  orc.random_matrix(4, 1, 6)[:, 0])
    core, us = orc.hosvd(flat(t), (5, 6, 4), 1e-10)
    assert [u.shape[1] for u in us] == [1, 1, 1]
    assert rel(flat(t), tucker_reconstruct(core, [1, 1, 1], *us)) < 1e-13
    t = orc.random_tensor(6, 6, 6, 7)
    core, us = orc.hosvd(t, (6, 6, 6), 0.0)
    assert [u.shape[1] for u in us] == [6, 6, 6]
    assert rel(t, tucker_reconstruct(core, [6, 6, 6], *us)) < 1e-13
    with pytest.raises(orc.OracleError):
        orc.hosvd(np.zeros(0, complex), (0, 2, 2), 1e-6)


def test_hosvd_energy_bound_and_orthonormal(orc):  # test_decomp.cpp:112-134
    for trial in range(5):
        dims = (8, 7, 9)
        core0 = orc.random_tensor(3, 2, 4, 1000 + 7 * trial)
        us0 = [np.linalg.qr(orc.random_matrix(dims[q], r, 1001 + 7 * trial + q))[0] for q, r in enumerate((3, 2, 4))]
        t = tucker_reconstruct(core0, (3, 2, 4), *us0)
        nz = orc.random_tensor(8, 7, 9, 1004 + 7 * trial)
        t = t + 1e-5 * np.linalg.norm(t) / np.linalg.norm(nz) * nz
        for tol in (1e-2, 1e-4, 1e-8):
            core, us = orc.hosvd(t, dims, tol)
            rk = [u.shape[1] for u in us]
            err = np.linalg.norm(tucker_reconstruct(core, rk, *us) - t)
            assert err <= tol * np.linalg.norm(t) * (1 + 1e-12)
            for u in us:
                assert np.allclose(u.conj().T @ u, np.eye(u.shape[1]), atol=1e-12)
