"""Device Green's-tensor assembly (vie_assemble, kernels_assembly.cu) against the oracle's
restatement of assembly.hpp / kernels.hpp / quadrature.hpp (pinned by the reference's
own assembly tests in tests/test_oracle_assembly.py), the reference's assembly known
answers run on the device (test_assembly.cpp), acceptance criterion 1 end to end on the
device (acceptance.cpp:41-83: assembled 3x3x4 N, compressed at tol 1e-10, against the dense
BTTB matrix and the dense FFT path over 20 seeded inputs, <= 1e-8), and the device
HOSVD's ranks against the oracle's QR + Jacobi SVD HOSVD at tight tolerances
(test_decomp.cpp:31-134)."""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

C0 = 299792458.0


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os

    import paper_1811_00484_b200 as vie

    O.set_threads(os.cpu_count() or 1)
    return vie, torch, vie.DftService(0)


def dev_asm(env, dims, res, k0, op, q, qp, quad=None):
    vie, torch, dft = env
    qs = vie.QuadratureSpec(*quad) if quad else None
    return vie.assemble_defining_tensor(dft, vie.VoxelGrid(dims, res), k0, op, q, qp, qs).cpu().numpy()


CASES = [((5, 4, 6), (0.01, 0.01, 0.01), 6.0), ((4, 7, 3), (0.002, 0.003, 0.0025), 2 * math.pi * 2.98e8 / C0 * 8.0),
         ((9, 2, 3), (0.01, 0.008, 0.012), 40.0)]


@pytest.mark.parametrize("dims,res,k0", CASES)
def test_device_assembly_matches_oracle(env, dims, res, k0):
    comps = [(0, q, qp) for q in range(3) for qp in range(q, 3)] + [(1, 0, 1), (1, 0, 2), (1, 1, 2), (2, 0, 0)]
    for op, q, qp in comps:
        t = dev_asm(env, dims, res, k0, op, q, qp)
        r = O.assemble(dims, res, k0, op, q, qp)
        err = np.max(np.abs(t - r)) / np.max(np.abs(r))
        assert err <= 1e-12, (op, q, qp, err)


def test_device_quadrature_budget_matches_oracle(env):
    quad = (3, 6, 2, 8, 4)
    t = dev_asm(env, (4, 4, 4), (0.01, 0.01, 0.01), 10.0, 0, 0, 2, quad)
    r = O.assemble((4, 4, 4), (0.01, 0.01, 0.01), 10.0, 0, 0, 2, quad)
    assert np.max(np.abs(t - r)) / np.max(np.abs(r)) <= 1e-12


def test_self_static_term_on_device(env):  # test_assembly.cpp:114-152
    vie, torch, dft = env
    dg, gram, err, conv = vie.self_static_term(dft, [1.0, 1.0, 1.0])
    depol = -dg / gram
    assert np.all(np.abs(depol - 1 / 3) <= 1e-6) and conv
    dg, gram, _, _ = vie.self_static_term(dft, [1.0, 1.5, 0.7])
    assert abs(np.sum(-dg / gram) - 1.0) <= 1e-8
    a, _, _, _ = vie.self_static_term(dft, [1.0, 1.0, 1.0])
    b, _, _, _ = vie.self_static_term(dft, [2.0, 2.0, 2.0])
    assert abs(b[0] / 8 - a[0]) <= 1e-12
    _, _, err, conv = vie.self_static_term(dft, [1.0, 1.0, 1.0], vie.QuadratureSpec(surface_points_per_axis=1))
    assert not conv and err > 1e-7
    ro = O.self_static_term([1.0, 1.5, 0.7])[0]
    assert np.max(np.abs(dg - ro)) <= 1e-13 * np.max(np.abs(ro))


def test_assembly_known_answers_on_device(env):  # test_assembly.cpp:166-216, 305-328
    vie, torch, dft = env
    res = (0.01, 0.01, 0.01)
    assert np.all(dev_asm(env, (3, 3, 3), res, 6.0, 1, 1, 1) == 0)
    xy, yx = dev_asm(env, (3, 2, 2), res, 6.0, 0, 0, 1), dev_asm(env, (3, 2, 2), res, 6.0, 0, 1, 0)
    assert np.linalg.norm(xy - yx) / np.linalg.norm(xy) < 1e-12
    kxy, kyx = dev_asm(env, (2, 2, 3), res, 6.0, 1, 0, 1), dev_asm(env, (2, 2, 3), res, 6.0, 1, 1, 0)
    assert np.linalg.norm(kxy + kyx) / np.linalg.norm(kxy) < 1e-12
    n3 = dev_asm(env, (3, 3, 3), res, 6.0, 0, 0, 1).reshape((3, 3, 3), order="F")
    k3 = dev_asm(env, (3, 3, 3), res, 6.0, 1, 0, 1).reshape((3, 3, 3), order="F")
    assert np.all(n3[0] == 0) and np.all(n3[:, 0] == 0) and np.all(k3[:, :, 0] == 0)
    dm, tw = 0.01, 2 * math.pi / 10
    t = dev_asm(env, (6, 1, 1), (dm, dm, dm), tw / dm, 0, 0, 0)
    ref = O.correlation_entry(0, tw, 0, 0, [5.0, 0.0, 0.0], [1.0, 1.0, 1.0], 16) * dm ** 3
    assert abs(t[5] - ref) / abs(ref) < 1e-8
    t = dev_asm(env, (1, 1, 1), res, 1e-3, 0, 2, 2)
    assert abs(t[0].real / 1e-6 - 2 / 3) <= 1e-6 and abs(t[0].imag) / 1e-6 < 1e-8
    g = dev_asm(env, (2, 1, 1), res, 1.0, 2, 0, 0)
    assert g[0].real > 0 and g[0].real > abs(g[1])
    with pytest.raises(ValueError):
        vie.assemble_defining_tensor(dft, vie.VoxelGrid((2, 2, 2), res), 1.0, 0, 0, 0, basis=vie.PWL)
    with pytest.raises(ValueError):
        vie.assemble_defining_tensor(dft, vie.VoxelGrid((2, 2, 2), res), 1.0, 0, 0, 0,
                                     vie.QuadratureSpec(far_points_per_axis=0))


def test_acceptance_criterion_1_on_device(env):  # acceptance.cpp:41-83
    vie, torch, dft = env
    dims, res = (3, 3, 4), (0.01, 0.01, 0.01)
    k0 = 2 * math.pi * 3e8 / C0
    grid = vie.VoxelGrid(dims, res)
    comps, par, _ = O.component_table(0, 0)
    # device: assemble -> tucker_compress (tol 1e-10, energy rule) -> operator
    tens = vie.assemble_operator(dft, grid, k0, vie.KIND_N)
    forms = [vie.tucker_compress(dft, t, dims, par[c], 1e-10) for c, (_, t) in enumerate(tens)]
    op = vie.build_operator_spectra(vie.KIND_N, vie.PWC, dims, [c for c, _ in tens], forms, dft)
    # oracle: the same assembly on the CPU -> dense BTTB matrix and the dense FFT path
    otens = [O.assemble(dims, res, k0, 0, int(c[0]), int(c[1])) for c in comps]
    dense = O.dense_bttb(0, 0, dims, otens)
    spectra = [O.dense_spectrum(t, dims, par[c]) for c, t in enumerate(otens)]
    nv = int(np.prod(dims))
    g = O.gauss_stream(2024, 20 * 3 * nv)
    worst = 0.0
    for trial in range(20):
        x = g[trial * 3 * nv:(trial + 1) * 3 * nv]
        res_all = [dense @ x, O.apply_operator_dense(0, 0, dims, spectra, x),
                   vie.apply_operator(op, torch.from_numpy(x).cuda()).cpu().numpy()]
        for a in range(3):
            for b in range(a + 1, 3):
                worst = max(worst, np.linalg.norm(res_all[a] - res_all[b]) / np.linalg.norm(res_all[a]))
    assert worst <= 1e-8, worst


def _geometric_tensor(dims, decay, seed):
    """Tucker tensor with geometrically decaying mode spectra (test_decomp.cpp:31-62 style)."""
    rng = np.random.default_rng(seed)
    r = min(dims)
    us = [np.linalg.qr(rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r)))[0] for n in dims]
    core = np.zeros((r, r, r), complex)
    for a in range(r):
        core[a, a, a] = decay ** a
    core += 1e-3 * decay ** (r / 2) * (rng.standard_normal((r, r, r)) + 1j * rng.standard_normal((r, r, r)))
    t = np.einsum("abc,ia,jb,kc->ijk", core, *us)
    return t.reshape(-1, order="F")


@pytest.mark.parametrize("tol", [1e-6, 1e-8, 1e-10])
def test_device_hosvd_ranks_match_oracle_at_tight_tolerances(env, tol):
    vie, torch, dft = env
    for dims, decay, seed in [((12, 10, 14), 0.3, 1), ((16, 16, 9), 0.15, 2), ((20, 13, 11), 0.5, 3)]:
        t = _geometric_tensor(dims, decay, seed)
        ranks_ref = [u.shape[1] for u in O.hosvd(t, dims, tol)[1]]
        f = vie.tucker_compress(dft, t, dims, (1, 1, 1), tol)
        assert tuple(f.ranks) == tuple(int(r) for r in ranks_ref), (dims, tol, f.ranks, ranks_ref)


@pytest.mark.parametrize("comp", [(0, 0, 0), (0, 0, 1), (0, 1, 2)])
def test_device_hosvd_ranks_on_assembled_tensors(env, comp):
    # the C5 path: an assembled component compressed on the device at tol 1e-4 .. 1e-10 has
    # the ranks of the oracle's QR + Jacobi SVD HOSVD (decomp.hpp:40-176)
    vie, torch, dft = env
    dims, res = (24, 20, 22), (0.005, 0.005, 0.005)
    k0 = 2 * math.pi * 2.98e8 / C0
    op, q, qp = comp
    t_dev = vie.assemble_defining_tensor(dft, vie.VoxelGrid(dims, res), k0, op, q, qp)
    t = O.assemble(dims, res, k0, op, q, qp)
    par = [1, 1, 1]
    if q != qp:
        par[q] = par[qp] = -1
    for tol in (1e-4, 1e-6, 1e-8, 1e-10):
        ranks_ref = [u.shape[1] for u in O.hosvd(t, dims, tol)[1]]
        f = vie.tucker_compress(dft, t_dev, dims, par, tol)
        assert tuple(f.ranks) == tuple(ranks_ref), (comp, tol, f.ranks, ranks_ref)
