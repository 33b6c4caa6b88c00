"""The drop-in boundary without a GPU.

* libtbf_b200.so loads and exports every function include/oiobf_b200.h
  declares (parsed from the header, so a new declaration without an export --
  or the reverse -- fails here);
* the Python mirror's EXPORTS list matches the header;
* host-only entry points (derive_seed, select_proxies_count, last_error) agree
  with the oracle; compute entry points fail loudly (no CPU fallback) when no
  device is present.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

from paper_2411_03029_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oiobf_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(re.findall(r"\b(oiobf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def test_header_declares_the_reference_path():
    fns = header_functions()
    for core in ("oiobf_tbf_construct", "oiobf_tbf_contract", "oiobf_tbf_memory", "oiobf_column_id_batch",
                 "oiobf_select_proxies_count", "oiobf_derive_seed", "oiobf_subtensor_at",
                 "oiobf_mode_product_blockdiag", "oiobf_tbf_contract_phase"):
        assert core in fns


def test_exports_list_matches_header():
    assert sorted(_lib.EXPORTS) == header_functions()


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    defined = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [f for f in header_functions() if f not in defined]
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points_match_oracle(lib, oracle):
    tags = np.array([0x56, 1, 2, 3, 0, 1, 0], np.uint64)
    for seed in (0, 1, 0xDEADBEEF, 2 ** 63 + 5):
        assert lib.oiobf_derive_seed(seed, tags, len(tags)) == oracle.derive_seed(seed, [int(t) for t in tags])
    for extent, count, mode in ((64, 8, 1), (1000, 37, 1), (5, 9, 1), (2 ** 20, 64, 1), (1000, 37, 2), (40, 3, 0)):
        out = np.zeros(extent if mode == 0 else max(count, 1), np.int64)
        n = np.zeros(1, np.int64)
        assert lib.oiobf_select_proxies_count(extent, count, mode, 77, out, n) == 0
        got = out[: n[0]]
        ref = oracle.select_proxies_count(extent, count, mode, 77)
        np.testing.assert_array_equal(got, ref)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_compute_fails_loudly_without_device(lib):
    import paper_2411_03029_b200 as tb
    from paper_2411_03029_b200.configs import green_plates
    with pytest.raises(Exception):
        tb.tbf_construct(green_plates(32), 2, 1e-6, seed=1)
    assert lib.oiobf_last_error()  # an error message is recorded, not a silent fallback


def test_new_entry_points_reject_bad_arguments(lib, tmp_path):
    """TBF1 load and the apply-engine selector validate their arguments before
    touching a device (std::invalid_argument -> OIOBF_EINVAL)."""
    import ctypes as C
    h = C.c_void_p()
    assert lib.oiobf_tbf_load(str(tmp_path / "missing.tbf1").encode(), C.byref(h)) == 1
    assert b"cannot open" in lib.oiobf_last_error()
    bad = tmp_path / "bad.tbf1"
    bad.write_bytes(b"NOPE" + bytes(64))
    assert lib.oiobf_tbf_load(str(bad).encode(), C.byref(h)) == 1
    assert b"not a TBF1 file" in lib.oiobf_last_error()
    assert lib.oiobf_tbf_set_apply_engine(None, 1) == 1
    assert lib.oiobf_tbf_save(None, b"x") == 1


def test_tbf1_header_reader_rejects_garbage(tmp_path):
    from paper_2411_03029_b200.tbf1 import read_header, read_tbf1
    p = tmp_path / "g.tbf1"
    p.write_bytes(b"TBF2" + bytes(200))
    with pytest.raises(ValueError):
        read_header(str(p))
    with pytest.raises(ValueError):
        read_tbf1(str(p))
