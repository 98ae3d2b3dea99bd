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


def test_plan_size_bound_and_owner_math():
    """The stream-K index math is 32-bit (rb_plan.h: total x grid < 2^32,
    larger plans rejected) and the device finds a tile's owner by a
    multiply-high with ceil(2^64 / total): restated here and checked against
    the exact division over the edge cases of the bound."""
    import pytest
    from paper_2402_14808_b200 import _lib
    from paper_2402_14808_b200.errors import DimensionError
    with pytest.raises(DimensionError):
        _lib.sys_plan(4096, 64, 64, 1 << 22, 148)   # 64 heads x 4.2M keys x 148 CTAs
    fields, _ = _lib.sys_plan(256, 64, 8, 65536, 148)
    assert fields["total"] * fields["grid"] < 1 << 32
    for total in (2, 3, 7, 127, 4096, 32768, 33554431, (1 << 32) // 148):
        magic = (2 ** 64 - 1) // total + 1
        for grid in (1, 90, 148):
            for x in (0, 1, total // 3, total - 2, total - 1):
                n = (x + 1) * grid - 1
                if n >= 1 << 32:
                    continue
                assert (n * magic) >> 64 == n // total, (total, grid, x)
