"""The C-ABI library loads on a CPU-only host and exports every symbol
include/ellwarp_b200.h declares. Only host-side entry points are called."""
import os
import re

import pytest

from paper_1501_00324_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ellwarp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(ew_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


def test_header_symbols_exported():
    lib = capi.lib()
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert sorted(capi.declared_symbols()) == declared()


def test_kernel_ids_and_support():
    # kernel_ids() order, kernels.cpp:7-12
    assert capi.kernel_ids() == ["csr_ref", "csr_vector", "coo", "ell", "hyb", "k1", "k1r", "k1rs", "k2",
                                 "k2r", "k2rs"]
    lib = capi.lib()
    for k in ("csr_ref", "k1", "k1r", "k1rs", "k2", "k2r", "k2rs"):
        assert lib.ew_kernel_id_supported(k.encode()) == 1
    assert lib.ew_kernel_id_supported(b"bogus") == -1
    assert lib.ew_abi_version() == 1


def test_host_only_entry_points(golden):
    for nnz, t, ws, want in golden["k2_lanes"]:
        assert capi.compute_k2_lanes(nnz, t, ws) == want
    with pytest.raises(ValueError):
        capi.compute_k2_lanes(5, 0, 32)
    with pytest.raises(ValueError):
        capi.compute_k2_lanes(5, 2, 12)
    assert capi.compute_alpha(10.0, 1.0, 2.0) == 10
    assert capi.compute_alpha(0.0, 3.0, 2.0) is None
    assert capi.compute_alpha(0.0, 1.0, 2.0) == 1
    with pytest.raises(ValueError):
        capi.compute_alpha(-1.0, 1.0, 2.0)


def test_no_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(capi, "_lib", None)
    monkeypatch.setattr(capi, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        capi.lib()
