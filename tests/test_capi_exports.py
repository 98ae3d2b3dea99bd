"""The C-ABI library loads and exports every symbol include/relay_b200.h
declares (no compute calls: no GPU needed)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header="relay_b200.h"):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int)\s+(rb_\w+)\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("rb_system_attention", "rb_context_attention", "rb_relay_fusion",
              "rb_kv_append", "rb_last_error", "rb_sys_plan_query"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2402_14808_b200 import _lib
    lib = _lib.load()
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(raw, name), name
    assert set(_declared()) == set(_lib.EXPORTS)
    assert lib.rb_abi_version() == _lib.ABI_VERSION
    # the diagnostics entry points are not part of the production ABI
    for name in _declared("relay_b200_diag.h"):
        assert not hasattr(raw, name), name


def test_diag_library_exports_both_headers():
    from paper_2402_14808_b200 import _lib
    if not os.path.exists(_lib.DIAG_LIB_PATH):
        import pytest
        pytest.skip("diagnostics build absent")
    raw = ctypes.CDLL(_lib.DIAG_LIB_PATH)
    assert set(_declared("relay_b200_diag.h")) == set(_lib.DIAG_EXPORTS)
    for name in _declared() + _declared("relay_b200_diag.h"):
        assert hasattr(raw, name), name


def test_error_mapping_without_gpu():
    import pytest
    from paper_2402_14808_b200 import _lib
    from paper_2402_14808_b200.errors import ContractError, DimensionError
    with pytest.raises(ContractError):
        _lib.sys_plan(4, 2, 2, 0, 148)          # empty system segment
    with pytest.raises(DimensionError):
        _lib.sys_plan(4, 3, 2, 16, 148)         # hq not a multiple of hkv
