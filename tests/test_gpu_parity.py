"""GPU parity: the B200 path (libvie_b200.so via the C ABI) against the CPU oracle
on identical seeded inputs.  Bar (BASELINE north star): matvec relative l2 error
<= 1e-10; GMRES iterations within +-1 and final residual within 1e-8."""
import numpy as np
import pytest

from tests.helpers import fourier_forms, random_field, rel, spatial_tucker_forms

pytestmark = pytest.mark.gpu

N, K, PWC, PWL = 0, 1, 0, 1
MATVEC_TOL = 1e-10  # north star: matvec relative l2 <= 1e-10


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


def make_ops(vie, dft, orc, kind, basis, dims, rank, seed, subset=None, scale=1.0):
    spatial, par = spatial_tucker_forms(kind, basis, dims, rank, seed)
    if scale != 1.0:
        spatial = [(core * scale, us) for core, us in spatial]
    comps, _, _ = vie.component_table(kind, basis)
    idx = list(range(len(comps))) if subset is None else list(subset)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in idx]
    op = vie.build_operator_spectra(kind, basis, dims, [comps[c] for c in idx], forms, dft)
    return op, fourier_forms(spatial, par), spatial, par


def to_dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_gpu(vie, op, x):
    import torch

    y = vie.apply_operator(op, to_dev(x))
    torch.cuda.synchronize()
    return y.cpu().numpy()


CASES = [
    (N, PWC, (3, 5, 4), 3), (K, PWC, (3, 5, 4), 3), (N, PWC, (4, 4, 4), 4), (N, PWC, (6, 5, 7), 5),
    (N, PWC, (1, 1, 2), 2), (N, PWC, (2, 3, 1), 2), (N, PWC, (8, 6, 10), 6), (K, PWC, (7, 9, 5), 4),
    (N, PWL, (3, 4, 5), 3), (K, PWL, (3, 4, 5), 3), (N, PWL, (2, 2, 2), 2), (N, PWL, (5, 3, 4), 4),
]


@pytest.mark.parametrize("kind,basis,dims,rank", CASES)
def test_matvec_matches_oracle(vie, dft, orc, kind, basis, dims, rank):
    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 7 + sum(dims))
    for trial in range(2):
        x = random_field(basis, dims, 2024 + trial)
        y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
        y = run_gpu(vie, op, x)
        assert rel(y_ref, y) <= MATVEC_TOL, (kind, basis, dims)


# n3 with a compile-time pencil shape (kernels_pencil2.cu: 32 = 4x8, 64 = 8x8, 100 = 10x10):
# odd/even axis-1 edges, partial last pair group (PWC packs 4 pairs per CTA), m1 = 2
# (edge launch only), both kinds and bases.
# Embedded lengths with a prime factor 11..31 on axes 1 / 2 (the Duke head's 186 = 6 x 31 and
# 238 = 14 x 17 are the motivation): the EXT two-stage row / column passes (fft.cuh prime
# DFTs).  Single-stage (22, 26, 34) and two-stage (62 = 2 x 31, 38, 46, 58, 186, 238) plans.
EXT_CASES = [
    (N, PWL, (11, 17, 6), 3), (K, PWC, (13, 19, 5), 3), (N, PWC, (31, 7, 8), 4), (N, PWL, (23, 29, 4), 3),
    (K, PWL, (19, 11, 32), 3), (N, PWL, (93, 13, 6), 4), (N, PWC, (7, 119, 5), 3),
    (N, PWL, (5, 3, 125), 3), (K, PWC, (6, 4, 125), 3),  # n3 = 125: odd axis-3 branch (generic pencil, the Duke grid)
]


@pytest.mark.parametrize("kind,basis,dims,rank", EXT_CASES)
def test_matvec_ext_prime_lengths(vie, dft, orc, kind, basis, dims, rank):
    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 5 + sum(dims))
    x = random_field(basis, dims, 77)
    y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
    y = run_gpu(vie, op, x)
    assert rel(y_ref, y) <= MATVEC_TOL, (kind, basis, dims)


def test_ext_prime_axis3_rejected(vie, dft, orc):
    """Axis 3 keeps the 7-smooth plans (pencil kernels): m3 = 2 x 17 is refused loudly."""
    with pytest.raises(ValueError):
        make_ops(vie, dft, orc, N, PWC, (4, 4, 17), 2, 3)


PENCIL2_CASES = [
    (N, PWL, (3, 4, 32), 3), (K, PWL, (4, 3, 100), 3), (N, PWC, (5, 3, 64), 4), (K, PWC, (6, 2, 32), 3),
    (N, PWC, (1, 2, 32), 2), (N, PWL, (7, 5, 64), 3), (N, PWC, (9, 4, 100), 3), (K, PWL, (2, 6, 64), 2),
    (N, PWL, (4, 3, 100), 3),  # the headline kernel k_pencil2<N, PWL, 10, 20>
]


@pytest.mark.parametrize("kind,basis,dims,rank", PENCIL2_CASES)
def test_matvec_pencil2_shapes(vie, dft, orc, kind, basis, dims, rank):
    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 11 + sum(dims))
    x = random_field(basis, dims, 77)
    y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
    assert rel(y_ref, run_gpu(vie, op, x)) <= MATVEC_TOL, (kind, basis, dims)


# PWL interior mirror groups on the DMMA-Hadamard kernel (kernels_pencil3.cu): n3 with a
# compiled shape (32 = 4x8, 64 = 8x8, 100 = 10x10, 128 = 8x16, 200 = 10x20), both kinds,
# interior groups in both axes, n2 = 2 (axis-2 edge rows only), n1 = 1 (axis-1 edge only)
PENCIL3_CASES = [
    (N, PWL, (5, 6, 32), 3), (K, PWL, (4, 5, 64), 3), (N, PWL, (3, 3, 128), 4), (K, PWL, (3, 4, 200), 3),
    (N, PWL, (6, 2, 100), 3), (N, PWL, (2, 7, 200), 5), (K, PWL, (1, 4, 64), 2), (N, PWL, (4, 5, 200), 25),
    (N, PWL, (3, 4, 48), 3), (K, PWL, (3, 3, 80), 2), (N, PWL, (4, 3, 96), 3), (K, PWL, (3, 3, 120), 2),
    (N, PWL, (3, 3, 160), 3), (N, PWC, (8, 3, 120), 3), (K, PWC, (8, 4, 96), 2),
]


@pytest.mark.parametrize("kind,basis,dims,rank", PENCIL3_CASES)
def test_matvec_pencil3_shapes(vie, dft, orc, kind, basis, dims, rank):
    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 13 + sum(dims))
    for trial in range(2):
        x = random_field(basis, dims, 91 + trial)
        y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
        assert rel(y_ref, run_gpu(vie, op, x)) <= MATVEC_TOL, (kind, basis, dims)


# strategy hosvd_loop: the fused persistent decompress x pencil kernel (kernels_fused.cu) with the
# spectrum tiles in an L2 ring.  Cases: every compiled axis-3 shape, both kinds, a tail tile
# (n1 - 1 not a multiple of 64), ring reuse (more tiles than ring slots), rank 25 and ranks that
# differ per mode.
LOOP_CASES = [
    (N, PWL, (5, 6, 32), 3), (K, PWL, (4, 5, 64), 3), (N, PWL, (3, 3, 128), 4), (K, PWL, (3, 4, 200), 3),
    (N, PWL, (3, 4, 48), 3), (K, PWL, (3, 3, 80), 2), (N, PWL, (4, 3, 96), 3), (K, PWL, (3, 3, 120), 2),
    (N, PWL, (3, 3, 160), 3),
    (N, PWL, (6, 2, 100), 3), (N, PWL, (70, 9, 32), 4), (K, PWL, (135, 3, 64), 2), (N, PWL, (4, 5, 200), 25),
]


@pytest.mark.parametrize("kind,basis,dims,rank", LOOP_CASES)
def test_matvec_hosvd_loop(vie, dft, orc, kind, basis, dims, rank):
    import torch

    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 17 + sum(dims))
    x = random_field(basis, dims, 93)
    y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
    y_dec = vie.apply_operator(op, to_dev(x), strategy="hosvd_decompress").cpu().numpy()
    ws_dec = op.workspace_bytes()
    y_loop = vie.apply_operator(op, to_dev(x), strategy="hosvd_loop").cpu().numpy()
    torch.cuda.synchronize()
    assert vie.get_strategy(op) == "hosvd_loop"
    assert rel(y_ref, y_loop) <= MATVEC_TOL, (kind, dims)
    assert rel(y_dec, y_loop) <= 1e-12, (kind, dims)
    assert op.workspace_bytes() > ws_dec  # both strategies' storage now allocated
    y_again = vie.apply_operator(op, to_dev(x), strategy="tucker_cp_loop").cpu().numpy()
    assert np.array_equal(y_again, y_loop)  # deterministic (fixed work order per tile)


def test_hosvd_loop_fresh_operator_holds_no_spectrum(vie, dft, orc):
    """A loop-only operator never allocates the whole-spectrum buffer: its workspace is below
    the decompress strategy's by about the octant spectra (NC (n1+1)(n2+1)(n3+1) x 16 B)."""
    dims = (40, 60, 32)  # 41 x 61 octant rows vs a 4 x 64-row ring + 200 edge rows
    op, oforms, _, _ = make_ops(vie, dft, orc, N, PWL, dims, 3, 5)
    vie.set_strategy(op, "hosvd_loop")
    x = random_field(PWL, dims, 3)
    y = vie.apply_operator(op, to_dev(x), strategy="hosvd_loop").cpu().numpy()
    assert rel(orc.apply_operator_tucker(N, PWL, dims, oforms, x), y) <= MATVEC_TOL
    op2, _, _, _ = make_ops(vie, dft, orc, N, PWL, dims, 3, 5)
    vie.apply_operator(op2, to_dev(x), strategy="hosvd_decompress")
    noct = 60 * 41 * 61 * 33 * 16
    assert op2.workspace_bytes() - op.workspace_bytes() >= 0.5 * noct


def test_hosvd_loop_unsupported_raises(vie, dft, orc):
    op, _, _, _ = make_ops(vie, dft, orc, N, PWC, (4, 4, 4), 2, 1)
    with pytest.raises(ValueError):
        vie.apply_operator(op, to_dev(random_field(PWC, (4, 4, 4), 1)), strategy="hosvd_loop")
    with pytest.raises(ValueError):
        vie.apply_operator(op, to_dev(random_field(PWC, (4, 4, 4), 1)), strategy="dense")


# kernel-path coverage: rank > 28 (FMA decompression fallback), an axis length without a
# two-stage plan (m = 250 = 2 x 5^3: generic multi-stage passes), and n3 without a compiled
# pencil shape (generic pencil kernel)
PATH_CASES = [
    (N, PWC, (6, 5, 7), 30),     # rank 30: k_decomp_s (FMA) instead of the DMMA kernel
    (N, PWC, (5, 4, 60), 100),   # rank 100 x n3 60: beyond the FMA tile, k_decomp_s_big
    (N, PWC, (125, 4, 3), 2),    # m1 = 250: generic row passes (three-stage plan)
    (N, PWL, (4, 125, 3), 2),    # m2 = 250: generic column passes
    (K, PWL, (3, 4, 9), 3),      # n3 = 9: no compiled pencil shape, generic pencil kernel
]


@pytest.mark.parametrize("kind,basis,dims,rank", PATH_CASES)
def test_matvec_kernel_paths(vie, dft, orc, kind, basis, dims, rank):
    op, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 31 + sum(dims))
    x = random_field(basis, dims, 5)
    y_ref = orc.apply_operator_tucker(kind, basis, dims, oforms, x)
    assert rel(y_ref, run_gpu(vie, op, x)) <= MATVEC_TOL, (kind, basis, dims, rank)


def test_matvec_c1_cube_pwl(vie, dft, orc):
    # BASELINE configs[0]: 32^3 PWL grid, r = 25 (CPU-runnable reference case)
    dims = (32, 32, 32)
    op, oforms, _, _ = make_ops(vie, dft, orc, N, PWL, dims, 25, 1234)
    x = random_field(PWL, dims, 2024)
    y_ref = orc.apply_operator_tucker(N, PWL, dims, oforms, x)
    assert rel(y_ref, run_gpu(vie, op, x)) <= MATVEC_TOL


def test_matvec_mixed_ranks_and_host_path(vie, dft, orc):
    dims = (6, 4, 5)
    spatial, par = spatial_tucker_forms(N, PWC, dims, 5, 99)
    rng = np.random.default_rng(0)
    mixed = []
    for c, (core, us) in enumerate(spatial):
        r = [1 + (c + q) % 5 for q in range(3)]
        g = (rng.standard_normal(r[0] * r[1] * r[2]) + 1j * rng.standard_normal(r[0] * r[1] * r[2]))
        mixed.append((g, [us[q][:, : r[q]] for q in range(3)]))
    comps, _, _ = vie.component_table(N, PWC)
    forms = [vie.TuckerForm(dft, dims, mixed[c][0], mixed[c][1], par[c]) for c in range(6)]
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    x = random_field(PWC, dims, 5)
    y_ref = orc.apply_operator_tucker(N, PWC, dims, fourier_forms(mixed, par), x)
    assert rel(y_ref, run_gpu(vie, op, x)) <= MATVEC_TOL
    assert rel(y_ref, vie.apply_operator(op, x)) <= MATVEC_TOL  # host-buffer C-ABI call


def test_host_batch_matches_single_calls(vie, dft, orc):
    # vie_matvec_host_batch: pipelined copies, results identical to one call per vector
    import torch

    dims = (5, 6, 4)
    op, oforms, _, _ = make_ops(vie, dft, orc, N, PWL, dims, 3, 5)
    xs = [random_field(PWL, dims, 40 + i) for i in range(5)]
    xp = [torch.from_numpy(x.copy()).pin_memory() for x in xs]
    yp = [torch.empty_like(x).pin_memory() for x in xp]
    vie.apply_operator_batch(op, xp, yp)
    for x, y in zip(xs, yp):
        assert np.array_equal(vie.apply_operator(op, x), y.numpy())
    assert rel(orc.apply_operator_tucker(N, PWL, dims, oforms, xs[3]), yp[3].numpy()) <= MATVEC_TOL
    assert vie.apply_operator_batch(op, []) == []


@pytest.mark.parametrize("basis", [PWC, PWL])
def test_component_sharding_sums_to_full(vie, dft, orc, basis):
    # components sharded over "ranks": partial outputs add up to the full matvec
    dims = (4, 3, 5)
    op, oforms, spatial, par = make_ops(vie, dft, orc, N, basis, dims, 3, 31)
    comps, _, _ = vie.component_table(N, basis)
    x = random_field(basis, dims, 3)
    full = run_gpu(vie, op, x)
    nc = len(comps)
    parts = []
    for r in range(3):
        sub = list(range(r, nc, 3))
        forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in sub]
        sop = vie.build_operator_spectra(N, basis, dims, [comps[c] for c in sub], forms, dft)
        parts.append(run_gpu(vie, sop, x))
    assert rel(full, sum(parts)) < 1e-13


def test_zero_input_gives_zero(vie, dft, orc):
    op, _, _, _ = make_ops(vie, dft, orc, N, PWC, (3, 3, 4), 2, 20)
    y = run_gpu(vie, op, np.zeros(3 * 36, complex))
    assert np.linalg.norm(y) == 0.0


@pytest.mark.parametrize("basis", [PWC, PWL])
def test_system_matvec_matches_oracle(vie, dft, orc, basis):
    import torch

    dims = (5, 4, 6) if basis == PWC else (3, 4, 3)
    op, oforms, _, _ = make_ops(vie, dft, orc, N, basis, dims, 3, 17)
    nv = int(np.prod(dims))
    rng = np.random.default_rng(4)
    eps = 1 + rng.uniform(0, 60, nv) - 1j * rng.uniform(0, 5, nv)
    inv_v = 0.37
    x = random_field(basis, dims, 20)
    y_ref = orc.apply_system_tucker(basis, dims, oforms, eps, inv_v, x)
    y = vie.apply_system(to_dev(eps), inv_v, op, to_dev(x))
    torch.cuda.synchronize()
    assert rel(y_ref, y.cpu().numpy()) <= MATVEC_TOL


def _scene(vie, dft, orc, basis, dims, seed):
    # synthetic spectra scaled so the system is a well-posed perturbation of M_eps
    # (oracle: PWC converges in ~17 iterations, PWL in ~66 with restarts)
    scale = 1e-4 if basis == PWC else 3e-5
    op, oforms, _, _ = make_ops(vie, dft, orc, N, basis, dims, 4, seed, scale=scale)
    nv = int(np.prod(dims))
    rng = np.random.default_rng(seed)
    eps = 1 + rng.uniform(1, 5, nv) - 1j * rng.uniform(0, 1, nv)
    rhs = random_field(basis, dims, seed + 1)
    return op, oforms, eps, rhs


@pytest.mark.parametrize("basis,dims", [(PWC, (6, 5, 4)), (PWL, (4, 3, 4))])
def test_gmres_matches_oracle(vie, dft, orc, basis, dims):
    op, oforms, eps, rhs = _scene(vie, dft, orc, basis, dims, 77)
    inv_v = 1.0
    ref = orc.gmres_system_tucker(basis, dims, oforms, eps, inv_v, rhs, tol=1e-8, inner=8, outer=20)
    res = vie.gmres(op, to_dev(eps), inv_v, to_dev(rhs), vie.GmresConfig(1e-8, 8, 20))
    assert ref.converged and res.converged
    assert abs(ref.iterations - res.iterations) <= 1
    assert abs(ref.final_relative_residual - res.final_relative_residual) <= 1e-8
    x = res.solution.cpu().numpy()
    ext = np.linalg.norm(orc.apply_system_tucker(basis, dims, oforms, eps, inv_v, x) - rhs) / np.linalg.norm(rhs)
    assert abs(ext - res.final_relative_residual) <= 1e-10
    assert rel(ref.solution, x) < 1e-6
    n = min(len(ref.residual_history), len(res.residual_history))
    assert np.allclose(ref.residual_history[:n], res.residual_history[:n], rtol=1e-6, atol=1e-12)


def test_gmres_zero_rhs_warm_start_and_nonconvergence(vie, dft, orc):
    dims = (4, 4, 3)
    op, oforms, eps, rhs = _scene(vie, dft, orc, PWC, dims, 5)
    z = vie.gmres(op, to_dev(eps), 1.0, to_dev(np.zeros_like(rhs)))
    assert z.converged and z.iterations == 0 and float(z.solution.abs().max()) == 0.0
    cold = vie.gmres(op, to_dev(eps), 1.0, to_dev(rhs), vie.GmresConfig(1e-10, 10, 10))
    assert cold.converged
    warm = vie.gmres(op, to_dev(eps), 1.0, to_dev(rhs), vie.GmresConfig(1e-10, 10, 10), x0=cold.solution)
    assert warm.converged and warm.iterations == 0
    bad = vie.gmres(op, to_dev(eps), 1.0, to_dev(rhs), vie.GmresConfig(1e-14, 1, 1))
    assert not bad.converged and bad.iterations == 1
    with pytest.raises(ValueError):
        vie.gmres(op, to_dev(eps), 1.0, to_dev(rhs), vie.GmresConfig(1e-5, 0, 1))
    nanr = rhs.copy()
    nanr[0] = np.nan
    with pytest.raises(ValueError):
        vie.gmres(op, to_dev(eps), 1.0, to_dev(nanr))


def test_error_behaviour(vie, dft, orc):
    dims = (3, 3, 3)
    spatial, par = spatial_tucker_forms(N, PWC, dims, 2, 3)
    comps, _, _ = vie.component_table(N, PWC)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(6)]
    with pytest.raises(ValueError):  # no components
        vie.build_operator_spectra(N, PWC, dims, [], [], dft)
    with pytest.raises(ValueError):  # duplicate component
        vie.build_operator_spectra(N, PWC, dims, [comps[0], comps[0]], [forms[0], forms[0]], dft)
    with pytest.raises(ValueError):  # not in the canonical table (K has no xx)
        vie.build_operator_spectra(K, PWC, dims, [comps[0]], [forms[0]], dft)
    with pytest.raises(ValueError):  # parity mismatch (form of xx used as xy)
        vie.build_operator_spectra(N, PWC, dims, [comps[1]], [forms[0]], dft)
    with pytest.raises(ValueError):  # inconsistent dims
        other = vie.TuckerForm(dft, (3, 3, 4), np.ones(1), [np.ones((3, 1)), np.ones((3, 1)), np.ones((4, 1))],
                               (1, 1, 1))
        vie.build_operator_spectra(N, PWC, dims, [comps[0]], [other], dft)
    with pytest.raises(ValueError):  # odd axis with a nonzero offset-0 row
        vie.TuckerForm(dft, dims, np.ones(1), [np.ones((3, 1)), np.ones((3, 1)), np.ones((3, 1))], (-1, -1, 1))
    with pytest.raises(ValueError):  # embedded length with a prime factor > 31 (2 * 37; 11..31 are served)
        f37 = vie.TuckerForm(dft, (37, 3, 3), np.ones(1), [np.ones((37, 1)), np.ones((3, 1)), np.ones((3, 1))],
                             (1, 1, 1))
        vie.build_operator_spectra(N, PWC, (37, 3, 3), [comps[0]], [f37], dft)
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    with pytest.raises(ValueError):
        vie.apply_operator(op, np.zeros(5, complex))
    with pytest.raises(ValueError):
        vie.apply_operator(op, np.zeros(81, complex), policy="no_buffer")


def test_fourier_domain_forms_accepted(vie, dft, orc):
    # domain=1: factors already transformed (transform_factors output, 2n rows)
    dims = (4, 5, 3)
    spatial, par = spatial_tucker_forms(N, PWC, dims, 3, 12)
    oforms = fourier_forms(spatial, par)
    comps, _, _ = vie.component_table(N, PWC)
    forms = [vie.TuckerForm(dft, dims, oforms[c].core, oforms[c].u, par[c], domain=1) for c in range(6)]
    op = vie.build_operator_spectra(N, PWC, dims, comps, forms, dft)
    x = random_field(PWC, dims, 8)
    assert rel(orc.apply_operator_tucker(N, PWC, dims, oforms, x), run_gpu(vie, op, x)) <= MATVEC_TOL


def test_linearity_at_head_2mm_size(vie, dft, orc):
    # size-independent property at BASELINE configs[2] shape (100x120x100, r=25)
    import torch

    dims = (100, 120, 100)
    op, _, _, _ = make_ops(vie, dft, orc, N, PWC, dims, 25, 42)
    n = 3 * int(np.prod(dims))
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    z = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    lam = 0.7 - 1.3j
    lhs = vie.apply_operator(op, x + lam * z)
    rhs = vie.apply_operator(op, x) + lam * vie.apply_operator(op, z)
    torch.cuda.synchronize()
    assert float((lhs - rhs).norm() / rhs.norm()) < 1e-12


def _embedded_value(core, ranks, us, par, d):
    """T~_c(d) of the circulant embedding (operator.hpp:40-74 / np_circulant_embed):
    t[|d|] per axis, times the axis parity for negative offsets; d: (P, 3) offsets."""
    g = np.asarray(core).reshape(tuple(ranks), order="F")
    rows = [us[q][np.abs(d[:, q]), :] * np.where(d[:, q] < 0, float(par[q]), 1.0)[:, None] for q in range(3)]
    return np.einsum("abg,pa,pb,pg->p", g, rows[0], rows[1], rows[2], optimize=True)


@pytest.mark.parametrize("kind,basis,s0,cell", [
    (N, PWL, 5, (17, 203, 99)), (N, PWL, 0, (199, 239, 199)), (N, PWL, 11, (0, 0, 0)),
    (K, PWL, 7, (120, 3, 150)), (N, PWC, 1, (5, 120, 198)), (K, PWC, 2, (199, 0, 77)),
])
def test_headline_size_delta_columns(vie, dft, orc, kind, basis, s0, cell):
    # BASELINE configs[1] shape (1 mm head grid 200x240x200, rank 25; the north star is
    # PWL N with 60 components): a unit current in cell r0 of current s0 returns column
    # (s0, r0) of the operator, y_t(r) = sum over blocks (t, s0, c, ds) of ds*sigma_c*T~_c(r - r0)
    # (operator.hpp:303-364), checked at 4096 sampled output cells of every target against
    # the Tucker forms evaluated directly.
    import torch

    dims = (200, 240, 200)
    rank = 25
    S = 12 if basis == PWL else 3
    spatial, par = spatial_tucker_forms(kind, basis, dims, rank, 7)
    comps, _, _ = vie.component_table(kind, basis)
    forms = [vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c]) for c in range(len(comps))]
    op = vie.build_operator_spectra(kind, basis, dims, comps, forms, dft)
    n1, n2, n3 = dims
    nv = n1 * n2 * n3
    x = torch.zeros(S * nv, dtype=torch.complex128, device="cuda")
    x[s0 * nv + cell[0] + n1 * (cell[1] + n2 * cell[2])] = 1.0
    y = vie.apply_operator(op, x)
    rng = np.random.default_rng(s0)
    pts = np.stack([rng.integers(0, n, 4096) for n in dims], axis=1)
    pts[:3] = [[0, 0, 0], [n1 - 1, n2 - 1, n3 - 1], list(cell)]
    flat_idx = pts[:, 0] + n1 * (pts[:, 1] + n2 * pts[:, 2])
    idx = torch.from_numpy(np.concatenate([t * nv + flat_idx for t in range(S)])).cuda()
    got = y[idx].cpu().numpy().reshape(S, -1)
    _, opar, blocks = orc.component_table(kind, basis)
    d = pts - np.asarray(cell)[None, :]
    want = np.zeros((S, len(pts)), np.complex128)
    cache = {}
    for t, s, c, ds in blocks:
        if s != s0:
            continue
        if c not in cache:
            cache[c] = _embedded_value(spatial[c][0], (rank,) * 3, spatial[c][1], opar[c], d)
        want[t] += ds * float(np.prod(opar[c])) * cache[c]
    assert np.linalg.norm(want) > 0
    assert rel(want, got) <= MATVEC_TOL, (kind, basis, s0, cell, rel(want, got))
