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
