"""Shared test helpers: seeded synthetic inputs in the reference's recipes and
an independent numpy restatement used to cross-check the C++ oracle.

The recipes follow /root/reference/proj/tests/test_fft_operator.cpp:17-42
(make_component_tensor / make_family / random_field) with seeds drawn from the
oracle's mt19937_64 + std::normal_distribution generator (test_util.hpp:9-31).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def flat(a3: np.ndarray) -> np.ndarray:
    """(n1, n2, n3) array -> reference flat layout i + n1*(j + n2*k)."""
    return np.asarray(a3).reshape(-1, order="F")


def unflat(v: np.ndarray, dims) -> np.ndarray:
    return np.asarray(v).reshape(tuple(dims), order="F")


def cp_reconstruct(f0, f1, f2) -> np.ndarray:
    """tensor.hpp:157-168 (returns flat)."""
    return flat(np.einsum("il,jl,kl->ijk", f0, f1, f2))


def tucker_reconstruct(core_flat, ranks, u1, u2, u3) -> np.ndarray:
    g = unflat(core_flat, ranks)
    return flat(np.einsum("abg,ia,jb,kg->ijk", g, u1, u2, u3, optimize=True))


def make_component_tensor(parity, dims, seed, rank=2) -> np.ndarray:
    """test_fft_operator.cpp:17-26: low-rank separable, parity-zero rows."""
    f = []
    for q in range(3):
        m = O.random_matrix(dims[q], rank, seed + 7 * q)
        if parity[q] < 0:
            m[0, :] = 0
        f.append(m)
    return cp_reconstruct(*f)


def make_family(kind, basis, dims, seed, rank=2):
    """test_fft_operator.cpp:28-36, over the (kind, basis) component table."""
    comps, par, _ = O.component_table(kind, basis)
    out = []
    s = seed
    for c in range(len(comps)):
        s += 1
        out.append(make_component_tensor(par[c], dims, s, rank))
    return out


def random_field(basis, dims, seed) -> np.ndarray:
    """test_fft_operator.cpp:38-42 (one random_tensor per current component)."""
    S = O.ncur(basis)
    nv = int(np.prod(dims))
    return np.concatenate([O.random_tensor(dims[0], dims[1], dims[2], seed + 100 * q) for q in range(S)])[: S * nv]


def spatial_tucker_forms(kind, basis, dims, rank, seed):
    """Synthetic spatial-domain Tucker forms: core and factors
    ~ CN(0,1), factor row 0 zeroed on odd axes; returns list of
    (core_flat, [U1,U2,U3] spatial (n_q, r)) plus the parity table."""
    comps, par, _ = O.component_table(kind, basis)
    forms = []
    for c in range(len(comps)):
        base = seed + 1000 * c
        core = O.gauss_stream(base, rank ** 3)
        us = []
        for q in range(3):
            u = O.random_matrix(dims[q], rank, base + 1 + q)
            if par[c][q] < 0:
                u[0, :] = 0
            us.append(u)
        forms.append((core, us))
    return forms, par


def fourier_forms(spatial, par):
    """transform_factors (operator.hpp:76-90) of each spatial form -> oracle Forms."""
    out = []
    for c, (core, us) in enumerate(spatial):
        uh = [O.transform_factor(us[q], int(par[c][q])) for q in range(3)]
        out.append(O.Form(core, uh[0], uh[1], uh[2]))
    return out


# ---- independent numpy restatement (cross-check of the C++ oracle) ----------
def np_circulant_embed(t_flat, dims, sign):
    n1, n2, n3 = dims
    t = unflat(t_flat, dims)
    e = np.zeros((2 * n1, 2 * n2, 2 * n3), np.complex128)
    def idx(n, s):
        src = np.concatenate([np.arange(n), [0], 2 * n - np.arange(n + 1, 2 * n)])
        sg = np.concatenate([np.ones(n), [0.0], np.full(n - 1, float(s))])
        return src, sg
    s1, g1 = idx(n1, sign[0])
    s2, g2 = idx(n2, sign[1])
    s3, g3 = idx(n3, sign[2])
    e = t[np.ix_(s1, s2, s3)] * g1[:, None, None] * g2[None, :, None] * g3[None, None, :]
    return flat(e)


def np_fft3(v_flat, dims, inverse=False):
    a = unflat(v_flat, dims)
    return flat(np.fft.ifftn(a) if inverse else np.fft.fftn(a))


def np_apply_dense(kind, basis, dims, tensors, x):
    comps, par, blocks = O.component_table(kind, basis)
    S = O.ncur(basis)
    n1, n2, n3 = dims
    nv = n1 * n2 * n3
    ed = (2 * n1, 2 * n2, 2 * n3)
    spectra = [np_fft3(np_circulant_embed(tensors[c], dims, par[c]), ed) for c in range(len(comps))]
    xh = []
    for s in range(S):
        pad = np.zeros(ed, np.complex128)
        pad[:n1, :n2, :n3] = unflat(x[s * nv:(s + 1) * nv], dims)
        xh.append(np_fft3(flat(pad), ed))
    yh = [np.zeros(int(np.prod(ed)), np.complex128) for _ in range(S)]
    for t, s, c, ds in blocks:
        sigma = float(np.prod(par[c]))
        yh[t] += ds * sigma * spectra[c] * xh[s]
    out = []
    for t in range(S):
        full = unflat(np_fft3(yh[t], ed, inverse=True), ed)
        out.append(flat(full[:n1, :n2, :n3]))
    return np.concatenate(out)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(a)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)
