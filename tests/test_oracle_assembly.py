"""The oracle's restatement of the Green's-tensor assembly (assembly.hpp, kernels.hpp,
quadrature.hpp) against the reference's own assembly tests (test_assembly.cpp), restated
test by test with the same inputs and tolerances.  CPU only."""
import math

import numpy as np
import pytest

from oracle import oracle as O

INV4PI = 1.0 / (4.0 * math.pi)
TENTH_WAVE = 2.0 * math.pi / 10.0  # k * delta at lambda/10 (test_assembly.cpp:11)


@pytest.fixture(autouse=True, scope="module")
def threads():
    import os

    O.set_threads(os.cpu_count() or 1)


def green(r, k):
    return O.kernel_eval(O.OP_G, k, 0, 0, r)


def test_green_static_limit_and_phase():  # test_assembly.cpp:40-53
    g = green([1.0, 0.0, 0.0], 0.0)
    assert abs(g.real - INV4PI) <= 1e-15 and g.imag == 0.0
    for k0 in (0.1, 2.0, 40.0):
        assert abs(abs(green([0.0, 1.0, 0.0], k0)) - INV4PI) <= 1e-15
    r = [0.3, -0.2, 0.9]
    assert green(r, 5.0) == green([-v for v in r], 5.0)


def test_green_singular_point_throws():  # test_assembly.cpp:55-57
    with pytest.raises(ValueError):
        green([0.0, 0.0, 0.0], 1.0)


def test_dynamic_radials():  # test_assembly.cpp:59-76
    k, R = 1.7, 2.3
    full = O.radial(R, k)
    dyn = O.radial(R, k, dynamic=True)
    assert abs(dyn[0] - (full[0] - INV4PI / R)) <= 1e-15
    assert abs(dyn[1] - (full[1] + INV4PI / R ** 2)) <= 1e-15
    assert abs(dyn[2] - (full[2] - 2 * INV4PI / R ** 3)) <= 1e-14
    k, R = 3.0, 1e-8
    dyn = O.radial(R, k, dynamic=True)
    assert abs(dyn[0].imag - (-k * INV4PI)) <= 1e-9
    assert abs(dyn[1].real - (-k * k * INV4PI / 2)) <= 1e-9
    assert abs(dyn[2].imag - (k ** 3 * INV4PI / 3)) <= 1e-8


def test_self_static_term():  # test_assembly.cpp:114-152
    dg, gram, err, conv = O.self_static_term([1.0, 1.0, 1.0])
    depol = -dg / gram
    assert np.all(np.abs(depol - 1.0 / 3.0) <= 1e-6) and conv
    assert abs(depol[0] - depol[1]) <= 1e-10 and abs(depol[1] - depol[2]) <= 1e-10
    dg, gram, _, _ = O.self_static_term([1.0, 1.5, 0.7])
    assert abs(np.sum(-dg / gram) - 1.0) <= 1e-8
    a, _, _, _ = O.self_static_term([1.0, 1.0, 1.0])
    b, _, _, _ = O.self_static_term([2.0, 2.0, 2.0])
    assert abs(b[0] / 8.0 - a[0]) <= 1e-12
    _, _, err, conv = O.self_static_term([1.0, 1.0, 1.0], quad=(5, 10, 1, 1, 6))
    assert not conv and err > 1e-7


def test_correlation_matches_brute_force_pair_integral():  # test_assembly.cpp:155-164
    dl = [1.0, 0.8, 1.2]
    d = [3.0 * dl[0], 2.0 * dl[1], 1.0 * dl[2]]
    brute = O.brute_pair_integral(O.OP_N, 0.4, 0, 1, d, dl, 10)
    corr = O.correlation_entry(O.OP_N, 0.4, 0, 1, d, dl, 8, False)
    assert abs(corr - brute) / abs(brute) < 1e-10


def test_k_diagonal_zero_and_direction_swaps():  # test_assembly.cpp:166-189
    res = (0.01, 0.01, 0.01)
    assert np.all(O.assemble((3, 3, 3), res, 6.0, O.OP_K, 1, 1) == 0)
    xy = O.assemble((3, 2, 2), res, 6.0, O.OP_N, 0, 1)
    yx = O.assemble((3, 2, 2), res, 6.0, O.OP_N, 1, 0)
    assert np.linalg.norm(xy - yx) / np.linalg.norm(xy) < 1e-12
    kxy = O.assemble((2, 2, 3), res, 6.0, O.OP_K, 0, 1)
    kyx = O.assemble((2, 2, 3), res, 6.0, O.OP_K, 1, 0)
    assert np.linalg.norm(kxy + kyx) / np.linalg.norm(kxy) < 1e-12


def test_parity_zeros_present():  # test_assembly.cpp:191-202
    res = (0.01, 0.01, 0.01)
    nxy = O.assemble((3, 3, 3), res, 6.0, O.OP_N, 0, 1).reshape((3, 3, 3), order="F")
    kxy = O.assemble((3, 3, 3), res, 6.0, O.OP_K, 0, 1).reshape((3, 3, 3), order="F")
    assert np.all(nxy[0, :, :] == 0) and np.all(nxy[:, 0, :] == 0) and np.all(kxy[:, :, 0] == 0)


def test_far_entry_matches_converged_oracle():  # test_assembly.cpp:204-216
    dm = 0.01
    t = O.assemble((6, 1, 1), (dm, dm, dm), TENTH_WAVE / dm, O.OP_N, 0, 0)
    ref = O.correlation_entry(O.OP_N, TENTH_WAVE, 0, 0, [5.0, 0.0, 0.0], [1.0, 1.0, 1.0], 16) * dm ** 3
    assert abs(t[5] - ref) / abs(ref) < 1e-8


def test_far_quadrature_converges_monotonically():  # test_assembly.cpp:218-229
    d, dl = [4.0, 1.0, 0.0], [1.0, 1.0, 1.0]
    ref = O.correlation_entry(O.OP_N, TENTH_WAVE, 0, 0, d, dl, 16)
    prev = math.inf
    for p in (2, 4, 8):
        err = abs(O.correlation_entry(O.OP_N, TENTH_WAVE, 0, 0, d, dl, p) - ref)
        assert err < prev
        prev = err


def test_far_entry_imaginary_part_vanishes_with_frequency():  # test_assembly.cpp:231-244
    entry = lambda k: O.correlation_entry(O.OP_N, k, 0, 0, [3.0, 0.0, 0.0], [1.0, 1.0, 1.0], 6)
    prev = abs(entry(0.5).imag)
    for k in (0.25, 0.125, 0.0625):
        im = abs(entry(k).imag)
        assert im < 0.75 * prev
        prev = im


def test_self_entry_static_limit():  # test_assembly.cpp:305-312
    t = O.assemble((1, 1, 1), (0.01, 0.01, 0.01), 1e-3, O.OP_N, 2, 2)
    v = 1e-6
    assert abs(t[0].real / v - 2.0 / 3.0) <= 1e-6 and abs(t[0].imag) / v < 1e-8


def test_scalar_kernel_self_entry_positive():  # test_assembly.cpp:314-319
    t = O.assemble((2, 1, 1), (0.01, 0.01, 0.01), 1.0, O.OP_G, 0, 0)
    assert t[0].real > 0 and t[0].real > abs(t[1])


def test_rejects_zero_budget():  # test_assembly.cpp:321-328 (PWL rejection is the C ABI's)
    with pytest.raises(ValueError):
        O.assemble((2, 2, 2), (0.01,) * 3, 1.0, O.OP_N, 0, 0, quad=(0, 10, 1, 12, 6))
