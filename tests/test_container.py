"""VIET container (container.hpp:15-159; tests restated from test_container.cpp:22-66) through
the library's C ABI (vie_container_*), pinned byte for byte against oracle/container.py.  Host
only: no GPU needed."""
import os

import numpy as np
import pytest

from oracle import container as ocont
from oracle import oracle as orc


@pytest.fixture(scope="module")
def vie():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1811_00484_b200 as v

    return v


def test_dense_round_trip_and_bytes(vie, tmp_path):
    t = orc.random_tensor(3, 4, 5, 1).reshape((3, 4, 5), order="F")  # test_container.cpp:22-30
    p = tmp_path / "vie_dense.bin"
    vie.save_container(p, t)
    back = vie.load_container(p)
    assert back.shape == (3, 4, 5) and np.array_equal(back, t)
    assert p.read_bytes() == ocont.encode(0, 0, 0.0, (3, 4, 5), (0, 0, 0), [t])
    assert vie.container_info(p) == {"kind": 0, "rule": 0, "tol": 0.0, "dims": (3, 4, 5), "ranks": (0, 0, 0)}


def test_tucker_round_trip_preserves_reconstruction(vie, tmp_path):
    dims = (6, 5, 4)
    t = orc.random_tensor(*dims, 2)  # test_container.cpp:32-45
    core, us = orc.hosvd(t, dims, 1e-6, rule=1)
    ranks = tuple(u.shape[1] for u in us)
    p = tmp_path / "vie_tucker.bin"
    vie.save_container(p, ("tucker", core.reshape(ranks, order="F"), us, 1, 1e-6))
    kind, c2, us2, rule, tol = vie.load_container(p)
    assert kind == "tucker" and rule == 1 and tol == 1e-6
    assert tuple(u.shape[1] for u in us2) == ranks
    assert all(np.array_equal(a, b) for a, b in zip(us, us2))
    assert np.array_equal(c2.reshape(-1, order="F"), core)
    assert p.read_bytes() == ocont.encode(1, 1, 1e-6, dims, ranks, list(us) + [core])
    # the restated reader agrees with the library writer
    k, r, tl, d, rk, payload = ocont.decode(p.read_bytes())
    assert (k, r, tl, d, rk) == (1, 1, 1e-6, dims, ranks) and payload.size == sum(
        dims[q] * ranks[q] for q in range(3)) + int(np.prod(ranks))


def test_tucker_cp_round_trip(vie, tmp_path):
    rng = np.random.default_rng(3)  # test_container.cpp:47-56 (CP factors given directly: no CP-ALS here)
    ws = [rng.standard_normal((5, 3)) + 1j * rng.standard_normal((5, 3)) for _ in range(3)]
    p = tmp_path / "vie_tcp.bin"
    vie.save_container(p, ("tucker_cp", ws))
    kind, ws2 = vie.load_container(p)
    assert kind == "tucker_cp" and all(np.array_equal(a, b) for a, b in zip(ws, ws2))
    assert p.read_bytes() == ocont.encode(2, 0, 0.0, (5, 5, 5), (3, 3, 3), ws)


def test_rejects_garbage_truncation_and_missing_files(vie, tmp_path):
    g = tmp_path / "vie_garbage.bin"  # test_container.cpp:58-66: std::runtime_error -> VIE_EIO
    g.write_bytes(b"not a container")
    for bad in (g, tmp_path / "vie_nonexistent.bin"):
        with pytest.raises(vie.VieError) as e:
            vie.load_container(bad)
        assert e.value.code == 5
    p = tmp_path / "trunc.bin"
    vie.save_container(p, orc.random_tensor(3, 3, 3, 4).reshape((3, 3, 3), order="F"))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(vie.VieError):
        vie.load_container(p)
    v = tmp_path / "badver.bin"
    v.write_bytes(b"VIET" + (2).to_bytes(4, "little") + bytes(60))
    with pytest.raises(vie.VieError, match="version"):
        vie.load_container(v)
    assert not os.path.exists(tmp_path / "vie_nonexistent.bin")
