"""The C-ABI library loads and exports every symbol include/relay_b200.h
declares (no compute calls: no GPU needed)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "relay_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int)\s+(rb_\w+)\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("rb_relay_step", "rb_system_attention", "rb_context_attention", "rb_relay_fusion",
              "rb_kv_append", "rb_last_error", "rb_step_plan_query"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2402_14808_b200 import _lib
    lib = _lib.load()
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(raw, name), name
    assert set(_declared()) == set(_lib.EXPORTS)
    assert lib.rb_abi_version() == _lib.ABI_VERSION == 3


def test_error_mapping_without_gpu():
    import pytest
    from paper_2402_14808_b200 import _lib
    from paper_2402_14808_b200.errors import ContractError, DimensionError
    lib = _lib.load()
    # empty system segment: the contract check runs before any device work
    st = lib.rb_relay_step(None, 0, 0, None, 1, 4, 1, 2, 2, 128, None, None, 0, 0, 0, None, None,
                           0, None, 0, 16, None, 0, 0, 0, None, 1, 0, 1.0, 148, None, 0, None,
                           None, 0, 3, None)
    with pytest.raises(ContractError):
        _lib.check(st, "rb_relay_step")
    with pytest.raises(DimensionError):
        _lib.step_plan(4, 3, 2, 16, 148)         # hq not a multiple of hkv
    assert _lib.relay_step_supported(32, 52, 52, 32, 16, True)
    assert not _lib.relay_step_supported(32, 12, 4, 32, 16, True)   # g = 3 does not divide nq
    assert not _lib.relay_step_supported(32, 8, 8, 32, 8, True)     # block size 8
