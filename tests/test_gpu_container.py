"""Device forms through the VIET container: a form built from spatial factors (tucker_compress
on the device, TuckerForm, tucker_cp_form) saved with vie_tucker_save and re-created with
vie_tucker_load (transform_factors on the device) gives the identical operator."""
import numpy as np
import pytest

from tests.helpers import random_field, rel
from tests.test_gpu_parity import N, PWC, PWL, dft, make_ops, vie  # noqa: F401

pytestmark = pytest.mark.gpu


def test_saved_forms_rebuild_the_same_operator(vie, dft, orc, tmp_path):
    import torch

    kind, basis, dims = N, PWL, (6, 5, 8)
    op, oforms, spatial, par = make_ops(vie, dft, orc, kind, basis, dims, 3, 12)
    comps, _, _ = vie.component_table(kind, basis)
    loaded = []
    for c in range(len(comps)):
        f = vie.TuckerForm(dft, dims, spatial[c][0], spatial[c][1], par[c])
        p = tmp_path / f"comp{c}.viet"
        vie.save_container(p, f)
        assert vie.container_info(p)["kind"] == 1
        loaded.append(vie.load_container(p, dft, par[c]))
    op2 = vie.build_operator_spectra(kind, basis, dims, comps, loaded, dft)
    x = torch.from_numpy(random_field(basis, dims, 5)).cuda()
    assert torch.equal(vie.apply_operator(op, x), vie.apply_operator(op2, x))


def test_device_compressed_and_cp_forms_round_trip(vie, dft, orc, tmp_path):
    import torch

    dims, sign = (9, 7, 8), (1, 1, 1)
    t = torch.from_numpy(orc.random_tensor(*dims, 3)).cuda()
    f = vie.tucker_compress(dft, t, dims, sign, tol=1e-6, rule=vie.RULE_ENERGY)
    p = tmp_path / "compressed.viet"
    vie.save_container(p, f)
    info = vie.container_info(p)
    assert info["kind"] == 1 and info["rule"] == 1 and info["tol"] == 1e-6 and info["ranks"] == tuple(f.ranks)
    kind_, core, us, rule, tol = vie.load_container(p)  # host tuple: the spatial factors
    assert kind_ == "tucker" and core.shape == tuple(f.ranks)
    g = vie.load_container(p, dft, sign)
    assert tuple(g.ranks) == tuple(f.ranks)
    rng = np.random.default_rng(4)
    ws = [rng.standard_normal((dims[q], 3)) + 1j * rng.standard_normal((dims[q], 3)) for q in range(3)]
    cp = vie.tucker_cp_form(dft, dims, ws, sign)
    q = tmp_path / "cp.viet"
    vie.save_container(q, cp)
    assert vie.container_info(q)["kind"] == 2
    kind2, ws2 = vie.load_container(q)
    assert kind2 == "tucker_cp" and all(np.array_equal(a, b) for a, b in zip(ws, ws2))
    assert tuple(vie.load_container(q, dft, sign).ranks) == (3, 3, 3)
