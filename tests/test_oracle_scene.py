"""Pins the oracle's solve_scene stages (build_rhs, recover_fields, postprocess;
solver.hpp:148-285) against the reference's own known-answer tests and an
independent numpy restatement (no GPU).  Paths relative to /root/reference/proj."""
import ctypes as C

import numpy as np
import pytest

EPS0, MU0, C0 = 8.8541878128e-12, 1.25663706212e-6, 299792458.0


def block_eps(dims, freq, eps, sigma):  # tests/test_solver.cpp:13-21 (block_map)
    e = np.ones(dims[::-1], np.complex128)  # [k][j][i] -> flat = i + n1 (j + n2 k)
    e[1:-1, 1:-1, 1:-1] = eps - 1j * sigma / (EPS0 * 2 * np.pi * freq)  # grid.hpp:72-74
    return e.reshape(-1)


def scene(dims, freq, res=0.01, origin=(0, 0, 0), pol=(1, 0, 0), d=(0, 0, 1), amp=1.0):
    return dict(dims=dims, resolution=(res,) * 3, origin=origin, frequency=freq, polarization=pol, direction=d,
                amplitude=amp)


def np_centres(sc):
    n1, n2, n3 = sc["dims"]
    k, j, i = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    r = [sc["origin"][a] + ((i, j, k)[a].reshape(-1) + 0.5) * sc["resolution"][a] for a in range(3)]
    return np.stack(r)


def np_phase(sc, r):
    d = np.asarray(sc["direction"], float)
    d = d / np.linalg.norm(d)
    k0 = 2 * np.pi * sc["frequency"] / C0
    return np.exp(-1j * k0 * np.tensordot(d, r, 1))


def np_build_rhs(sc, eps):  # solver.hpp:152-179, centre sampling
    p = np.asarray(sc["polarization"], float)
    p = p / np.linalg.norm(p)
    ce = 1j * 2 * np.pi * sc["frequency"] * EPS0
    chi = eps - 1
    ph = np_phase(sc, np_centres(sc))
    return np.concatenate([np.where(chi != 0, ce * chi * p[q] * sc["amplitude"] * ph, 0) for q in range(3)])


def test_rhs_zero_contrast_is_zero(orc):  # test_solver.cpp:115-121
    sc = scene((3, 3, 3), 3e8)
    assert np.linalg.norm(orc.build_rhs(sc, np.ones(27, np.complex128))) == 0.0


def test_rhs_single_voxel_direct_substitution(orc):  # test_solver.cpp:123-132
    sc = scene((1, 1, 1), 3e8, origin=(-0.005, -0.005, -0.005))
    r = orc.build_rhs(sc, np.array([2.0 + 0j]))
    ce = 1j * 2 * np.pi * 3e8 * EPS0
    assert abs(r[0] - ce) < 1e-12 * abs(ce) and r[1] == 0 and r[2] == 0


def test_rhs_linear_in_amplitude(orc):  # test_solver.cpp:134-139
    eps = block_eps((4, 4, 4), 3e8, 4.0, 0.1)
    a = orc.build_rhs(scene((4, 4, 4), 3e8), eps)
    b = orc.build_rhs(scene((4, 4, 4), 3e8, amp=2.5), eps)
    assert np.linalg.norm(b - 2.5 * a) / np.linalg.norm(b) < 1e-14


def test_rhs_gauss_variant_consistent(orc):  # test_scene_io.cpp:141-161
    sc = scene((3, 3, 3), 2.98e8)
    eps = np.full(27, 5.0 - 1j * 0.2 / (EPS0 * 2 * np.pi * 2.98e8))
    c, g3, g5 = (orc.build_rhs(sc, eps, q) for q in (1, 3, 5))
    dc = np.linalg.norm(c - g3) / np.linalg.norm(g3)
    assert 1e-7 < dc < 1e-3
    assert np.linalg.norm(g5 - g3) / np.linalg.norm(g5) < 1e-12


def test_rhs_matches_numpy_oblique_wave(orc):
    sc = scene((5, 4, 3), 1.28e8, res=0.004, origin=(-0.01, 0.002, 0.03), pol=(0, 1, -1), d=(0, 1, 1), amp=3.0)
    rng = np.random.default_rng(3)
    eps = 1 + rng.standard_normal(60) + 1j * rng.standard_normal(60)
    eps[::7] = 1.0
    r = orc.build_rhs(sc, eps)
    assert np.linalg.norm(r - np_build_rhs(sc, eps)) <= 1e-14 * np.linalg.norm(r)


def test_plane_wave_must_be_orthogonal(orc):  # grid.hpp:86-87
    with pytest.raises(Exception, match="orthogonal"):
        orc.build_rhs(scene((2, 2, 2), 3e8, pol=(1, 0, 1)), np.ones(8, np.complex128))


def test_recover_zero_current_gives_incident_fields(orc):  # test_solver.cpp:218-246 (K j = 0)
    sc = scene((3, 3, 3), 3e8)
    eps = block_eps((3, 3, 3), 3e8, 4.0, 0.1)
    j = np.zeros(81, np.complex128)
    e, h = orc.recover_fields(sc, eps, j, kj=np.zeros(81, np.complex128))
    r = np_centres(sc)
    ph = np_phase(sc, r)
    scat = np.tile(eps != 1, 3)
    e_inc = np.concatenate([ph, 0 * ph, 0 * ph])  # pol = x
    assert np.max(np.abs(e - np.where(scat, 0, e_inc))) < 1e-14
    eta0 = np.sqrt(MU0 / EPS0)
    h_inc = np.concatenate([0 * ph, ph / eta0, 0 * ph])  # z x x = y
    assert np.max(np.abs(h - h_inc)) < 1e-14


def test_recover_e_inverts_current_definition(orc):  # test_solver.cpp:248-262
    sc = scene((4, 4, 4), 2.98e8)
    eps = block_eps((4, 4, 4), 2.98e8, 10.0, 0.5)
    j = np.concatenate([orc.random_tensor(4, 4, 4, 40 + q) for q in range(3)])
    e, h = orc.recover_fields(sc, eps, j)
    assert h is None
    ce = 1j * 2 * np.pi * 2.98e8 * EPS0
    chi = np.tile(eps - 1, 3)
    m = chi != 0
    assert np.all(np.abs(e[m] - j[m] / (ce * chi[m])) <= 1e-14 * np.abs(j[m] / (ce * chi[m])))


def test_postprocess_matches_definition(orc):  # solver.hpp:258-284
    sc = scene((4, 3, 5), 3e8, res=0.002)
    rng = np.random.default_rng(5)
    eps = block_eps((4, 3, 5), 3e8, 50.0, 0.7)
    e = rng.standard_normal(180) + 1j * rng.standard_normal(180)
    h = rng.standard_normal(180) + 1j * rng.standard_normal(180)
    p, tot, b1 = orc.postprocess(sc, eps, e, h)
    sigma = -eps.imag * EPS0 * 2 * np.pi * 3e8
    p_np = 0.5 * sigma * (np.abs(e.reshape(3, -1)) ** 2).sum(0)
    assert np.allclose(p, p_np, rtol=1e-14, atol=0)
    assert abs(tot - p_np.sum() * 0.002 ** 3) <= 1e-14 * abs(tot)
    hh = h.reshape(3, -1)
    assert np.allclose(b1, MU0 * np.abs(hh[0] + 1j * hh[1]), rtol=1e-14, atol=0)
    assert np.all(p[eps == 1] == 0)  # vacuum absorbs nothing


def test_scene_abi_validates_without_gpu():
    """The C ABI checks the scene before touching the device (no GPU here)."""
    import paper_1811_00484_b200.vie as v

    L = v.lib()
    sc = v._scene(v.DielectricMap(v.VoxelGrid((2, 2, 2), (0.01,) * 3), None, 3e8), v.PlaneWave((1, 0, 1)))
    buf = (C.c_double * 48)()
    assert L.vie_build_rhs(None, C.byref(sc), buf, 1, buf, None) == v.VIE_EINVAL
    assert b"orthogonal" in L.vie_last_error()
    sc = v._scene(v.DielectricMap(v.VoxelGrid((2, 0, 2), (0.01,) * 3), None, 3e8), v.PlaneWave())
    assert L.vie_postprocess(None, C.byref(sc), buf, buf, None, buf, None, None, None) == v.VIE_EINVAL
    sc = v._scene(v.DielectricMap(v.VoxelGrid((2, 2, 2), (0.01,) * 3), None, 3e8), v.PlaneWave())
    assert L.vie_build_rhs(None, C.byref(sc), buf, 0, buf, None) == v.VIE_EINVAL
