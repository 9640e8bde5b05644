"""Device GMRES (vie_gmres / vie_gmres_solve) against the oracle's restatement of
solver.hpp:34-142 on the reference's own GMRES known-answer tests
(test_solver.cpp:31-114, test_scene_io.cpp:107-139), plus the right preconditioner
(solver.hpp:74, :131) and the caller-stream ordering of vie_gmres_solve."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1811_00484_b200 as vie

    return vie, torch, vie.DftService(0)


def dense_pair(torch, a):
    """The same dense map for the device solver (torch) and the oracle (numpy)."""
    at = torch.from_numpy(a).cuda()
    return (lambda x, y: y.copy_(at @ x)), (lambda v: a @ v)


def diag_pair(torch, d):
    dt = torch.from_numpy(d).cuda()
    return (lambda x, y: y.copy_(dt * x)), (lambda v: d * v)


def col(m):
    return np.ascontiguousarray(m[:, 0])


def test_identity_one_iteration(env):  # test_solver.cpp:31-38
    vie, torch, dft = env
    rhs = col(orc.random_matrix(20, 1, 1))
    r = vie.gmres_map(dft, lambda x, y: y.copy_(x), torch.from_numpy(rhs).cuda())
    assert r.converged and r.iterations == 1
    assert np.linalg.norm(r.solution.cpu().numpy() - rhs) / np.linalg.norm(rhs) < 1e-12


def test_diagonal_matches_direct_solve(env):  # test_solver.cpp:40-53
    vie, torch, dft = env
    d = np.array([complex(i + 1.0, 0.5 * i) for i in range(10)])
    rhs = col(orc.random_matrix(10, 1, 2))
    dev, _ = diag_pair(torch, d)
    r = vie.gmres_map(dft, dev, torch.from_numpy(rhs).cuda(), vie.GmresConfig(1e-12))
    ex = rhs / d
    assert r.converged
    assert np.linalg.norm(r.solution.cpu().numpy() - ex) / np.linalg.norm(ex) < 1e-10


@pytest.mark.parametrize("seed,shift,inner,outer,tol", [(3, "spd", 5, 100, 1e-9), (5, 6.0, 25, 1, 1e-14),
                                                        (7, 5.0, 50, 200, 1e-8)])
def test_dense_systems_match_oracle(env, seed, shift, inner, outer, tol):  # test_solver.cpp:55-97
    vie, torch, dft = env
    n = {3: 30, 5: 25, 7: 20}[seed]
    a = orc.random_matrix(n, n, seed)
    a = a @ a.conj().T / n + 4 * np.eye(n) if shift == "spd" else a + shift * np.eye(n)
    rhs = col(orc.random_matrix(n, 1, seed + 1))
    dev, host = dense_pair(torch, a)
    r = vie.gmres_map(dft, dev, torch.from_numpy(rhs).cuda(), vie.GmresConfig(tol, inner, outer))
    ref = orc.gmres(host, rhs, tol=tol, inner=inner, outer=outer)
    assert r.iterations == ref.iterations and r.converged == ref.converged
    h, hr = np.array(r.residual_history), np.array(ref.residual_history)
    assert np.all(np.abs(h - hr) <= 1e-8 * hr + 1e-15)  # the two matmuls round differently
    for i in range(1, len(h)):  # monotone within a cycle (test_solver.cpp:70-82)
        if i % inner:
            assert h[i] <= h[i - 1] * (1 + 1e-12)
    ext = np.linalg.norm(a @ r.solution.cpu().numpy() - rhs) / np.linalg.norm(rhs)
    assert abs(ext - r.final_relative_residual) <= 1e-10 * max(1.0, ext)


def test_nonconvergence_is_a_flag(env):  # test_solver.cpp:99-114
    vie, torch, dft = env
    a = np.zeros((40, 40), complex)
    for i in range(39):
        a[i + 1, i] = 1.0
    a[0, 39] = 1.0
    rhs = np.zeros(40, complex)
    rhs[0] = 1.0
    dev, _ = dense_pair(torch, a)
    r = vie.gmres_map(dft, dev, torch.from_numpy(rhs).cuda(), vie.GmresConfig(1e-12, 3, 2))
    assert not r.converged and r.solution.numel() == 40
    bad = rhs.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        vie.gmres_map(dft, dev, torch.from_numpy(bad).cuda())


def test_warm_start_and_right_preconditioner(env):  # test_scene_io.cpp:107-139
    vie, torch, dft = env
    d8 = np.array([complex(2.0 + i, 0.3) for i in range(8)])
    rhs8 = torch.from_numpy(col(orc.random_matrix(8, 1, 1))).cuda()
    dev8, _ = diag_pair(torch, d8)
    cold = vie.gmres_map(dft, dev8, rhs8, vie.GmresConfig(1e-10))
    warm = vie.gmres_map(dft, dev8, rhs8, vie.GmresConfig(1e-10), x0=cold.solution)
    assert cold.converged and warm.converged and warm.iterations == 0
    d12 = np.array([complex(1.0 + 3.0 * i, -0.5 * i) for i in range(12)])
    rhs12 = torch.from_numpy(col(orc.random_matrix(12, 1, 2))).cuda()
    dev12, _ = diag_pair(torch, d12)
    inv = torch.from_numpy(1.0 / d12).cuda()
    for pre in (inv, lambda x, y: y.copy_(x * inv)):  # diagonal form and callback form
        r = vie.gmres_map(dft, dev12, rhs12, vie.GmresConfig(1e-12), precond=pre)
        assert r.converged and r.iterations == 1
        res = torch.from_numpy(d12).cuda() * r.solution - rhs12
        assert float(torch.linalg.vector_norm(res) / torch.linalg.vector_norm(rhs12)) < 1e-12


def _zero_pwl_op(vie, dft, grid):
    comps, par, _ = vie.component_table(0, 1)
    r = 2
    forms = [vie.TuckerForm(dft, grid, np.zeros(r ** 3), [np.zeros((n, r)) for n in grid], par[c])
             for c in range(len(comps))]
    return vie.build_operator_spectra(0, 1, grid, comps, forms, dft)


def test_system_solve_with_diagonal_preconditioner(env):
    # N = 0: apply_system = diag(eps g), so M = diag(1 / (eps g)) converges in one iteration
    vie, torch, dft = env
    grid = (6, 5, 4)
    nv = int(np.prod(grid))
    op = _zero_pwl_op(vie, dft, grid)
    eps = torch.from_numpy(2.0 + 0.01 * np.arange(nv) - 0.4j).cuda()
    g = torch.tensor([1.0 if s % 4 == 0 else 1.0 / 12.0 for s in range(12)], dtype=torch.complex128).cuda()
    m = (1.0 / (eps[None, :] * g[:, None])).reshape(-1)
    rhs = torch.randn(12 * nv, dtype=torch.complex128, device="cuda")
    plain = vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(1e-12, 50, 4))
    pc = vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(1e-12, 50, 4), precond=m)
    assert pc.converged and pc.iterations == 1 and plain.iterations > 1
    assert float(torch.linalg.vector_norm(plain.solution - pc.solution) / torch.linalg.vector_norm(pc.solution)) < 1e-10


def test_solve_orders_after_the_callers_stream(env):
    # rhs produced on a side stream: the solve must wait for it (vie_gmres_solve stream arg)
    vie, torch, dft = env
    grid = (8, 6, 5)
    nv = int(np.prod(grid))
    op = _zero_pwl_op(vie, dft, grid)
    eps = torch.full((nv,), 3.0 - 0.2j, dtype=torch.complex128, device="cuda")
    src = torch.randn(12 * nv, dtype=torch.complex128, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)  # ~10 ms of device time before the rhs is written
        rhs = src * 2.0
        r = vie.gmres(op, eps, 1.0, rhs, vie.GmresConfig(1e-12, 50, 4), stream=side.cuda_stream)
    side.synchronize()
    assert r.converged
    gfac = torch.tensor([1.0 if s % 4 == 0 else 1.0 / 12.0 for s in range(12)], dtype=torch.complex128).cuda()
    expect = (src * 2.0).reshape(12, nv) / (eps[None, :] * gfac[:, None])
    assert float(torch.linalg.vector_norm(r.solution - expect.reshape(-1)) / torch.linalg.vector_norm(expect)) < 1e-10
