"""CPU-side checks of the drop-in boundary: the sm_100a library builds, loads
without a GPU and exports every entry point include/vie_b200.h declares; the
product's component tables equal the oracle's; errors need no device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    from paper_1811_00484_b200 import vie

    return vie


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "vie_b200.h")).read()
    return sorted(set(re.findall(r"\b(vie_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(lib):
    L = lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s


def test_library_is_sm100a(lib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("basis", [0, 1])
def test_product_tables_equal_oracle(lib, orc, kind, basis):
    a = lib.component_table(kind, basis)
    b = orc.component_table(kind, basis)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_errors_without_gpu(lib):
    L = lib.lib()
    assert L.vie_matvec(None, None, None, None) == lib.VIE_EINVAL
    assert b"null" in L.vie_last_error()
    h = C.c_void_p()
    rc = L.vie_ctx_create(C.byref(h), 0)
    assert rc != 0  # no CUDA device in this container
    assert L.vie_component_table(5, 0, None, None, None, None, None) == lib.VIE_EINVAL
