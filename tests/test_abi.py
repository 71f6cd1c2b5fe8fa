"""The C-ABI library (-m "not gpu"): it loads, exports every symbol include/aknn.h
declares, and its host-only logic (alpha tables, argument validation, error
strings) behaves as documented.  No compute call needs a GPU here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle.oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "aknn.h")


@pytest.fixture(scope="module")
def ak():
    import __graft_entry__
    __graft_entry__._load_builder().build()
    import paper_1902_09465_b200 as m
    return m


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aknn_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("aknn_build", "aknn_build_shard", "aknn_query", "aknn_query_async",
                 "aknn_exact", "aknn_free", "aknn_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol(ak):
    out = subprocess.run(["nm", "-D", "--defined-only", ak.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(ak.EXPORTS) >= set(_declared())


def test_library_is_sm100a_code(ak):
    out = subprocess.run(["cuobjdump", "--list-elf", ak.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,d,delta", [(1000, 256, 0.05), (60000, 784, 0.05),
                                       (100000, 12288, 0.05), (8_000_000, 768, 0.01)])
def test_product_alpha_table_equals_oracle_table(ak, n, d, delta):
    """The library's own alpha builder (used when the caller passes NULL) produces the
    same fp64 bits as the oracle's table, which the parity tests pass explicitly."""
    assert np.array_equal(ak.alpha_table(n, delta, d, "theory"), orc.alpha_theory(n, delta, d))
    for c in (1.0, 0.1, 0.01):
        assert np.array_equal(ak.alpha_table(n, delta, d, "experimental", c),
                              orc.alpha_experimental(n, delta, d, c))


def test_alpha_table_domain_errors(ak):
    with pytest.raises(ak.AknnError) as e:
        ak.alpha_table(1, 0.5, 8, "theory")
    assert e.value.status == ak.AKNN_EINVAL
    with pytest.raises(ak.AknnError):
        ak.alpha_table(10, 1.5, 8, "experimental")


def test_strerror_names_every_status(ak):
    for s in (0, -1, -2, -3, -4, -5):
        assert ak._lib.aknn_strerror(s).startswith(b"AKNN_")


def test_build_validates_before_touching_the_device(ak):
    """EINVAL for n < 2 or d outside [1, 33025] is decided on the host."""
    h = C.c_void_p()
    x = np.zeros((1, 4), np.uint8)
    assert ak._lib.aknn_build(x.ctypes.data, 1, 4, C.byref(h)) == ak.AKNN_EINVAL
    x = np.zeros((4, 1), np.uint8)
    assert ak._lib.aknn_build(x.ctypes.data, 4, 0, C.byref(h)) == ak.AKNN_EINVAL
    assert ak._lib.aknn_build(x.ctypes.data, 4, 40000, C.byref(h)) == ak.AKNN_EINVAL
    assert b"outside" in ak._lib.aknn_last_error()


def test_query_validates_null_index(ak):
    res = ak.Result()
    assert ak._lib.aknn_query(None, None, 1, 1, 1, 0.05, 0, None, C.byref(res)) == ak.AKNN_EINVAL
