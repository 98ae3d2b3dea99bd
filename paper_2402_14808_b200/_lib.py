"""ctypes binding of librelay_b200.so (the C-ABI in include/relay_b200.h).

There is exactly one backend: the in-tree CUDA library.  If it is missing,
importing this module raises -- there is no CPU fallback (the float64 CPU
restatement under oracle/ is test infrastructure only).
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractError, DimensionError, KernelError

_HERE = os.path.dirname(os.path.abspath(__file__))
# RB_LIB: diagnostics only (a variant build of the same sources, see build.py)
# RB_DIAG=1: the diagnostics build (kernels with %globaltimer stamps)
DIAG_LIB_PATH = os.path.join(_HERE, "librelay_b200_diag.so")
LIB_PATH = os.environ.get("RB_LIB") or (
    DIAG_LIB_PATH if os.environ.get("RB_DIAG") == "1" else os.path.join(_HERE, "librelay_b200.so"))

RB_OK, RB_ERR_DIMENSION, RB_ERR_CONTRACT, RB_ERR_CUDA = 0, 1, 2, 3
ABI_VERSION = 4

# every symbol include/relay_b200.h declares
EXPORTS = (
    "rb_last_error", "rb_abi_version", "rb_device_sm_count", "rb_sys_plan_query",
    "rb_system_attention", "rb_context_attention", "rb_context_workspace_bytes",
    "rb_relay_fusion", "rb_kv_append",
    "rb_relay_workspace_bytes", "rb_relay_sys_grid", "rb_relay_attention",
    "rb_rope_rows", "rb_rope_append",
)
# include/relay_b200_diag.h: exported by librelay_b200_diag.so only
DIAG_EXPORTS = ("rb_debug_umma_probe", "rb_debug_set_timestamps")

_lib = None
_diag = None


def load():
    global _lib
    if _lib is None:
        _lib = _bind(LIB_PATH)
    return _lib


def load_diag():
    """The diagnostics build (layout probe, per-CTA timestamps)."""
    global _diag
    if _diag is None:
        _diag = _bind(DIAG_LIB_PATH)
        vp, i32 = ctypes.c_void_p, ctypes.c_int
        _diag.rb_debug_umma_probe.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp]
        _diag.rb_debug_set_timestamps.argtypes = [vp]
        for name in DIAG_EXPORTS:
            getattr(_diag, name).restype = i32
    return _diag


def _bind(path):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built; run `python -m paper_2402_14808_b200.build` "
            "(no CPU fallback exists for the relay path)")
    lib = ctypes.CDLL(path)
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_float
    fp = ctypes.POINTER(ctypes.c_float)
    lib.rb_last_error.restype = ctypes.c_char_p
    lib.rb_last_error.argtypes = []
    lib.rb_abi_version.restype = i32
    lib.rb_device_sm_count.argtypes = [i32, ctypes.POINTER(i32)]
    lib.rb_sys_plan_query.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(i64),
                                      ctypes.POINTER(ctypes.c_size_t)]
    lib.rb_system_attention.argtypes = [
        vp, i64, i64, i32, i32, i32, i32, vp, vp, i32, i64, i64, f32, i32, vp, vp, vp,
        ctypes.c_size_t, vp]
    lib.rb_context_attention.argtypes = [
        vp, i64, i64, vp, i32, i32, i32, i32, i32, i32,  # q .. d
        vp, vp, vp, i32, i32, vp, i64, i64, i64, vp,     # k .. ctx_lens
        i32, vp, vp, i32, i64, i64,                      # causal, prefix
        vp, vp, f32, vp, i32, vp,                        # o_sys .. lse_out
        i32, vp, ctypes.c_size_t, vp]                    # max_ctx_len, workspace, stream
    lib.rb_context_workspace_bytes.argtypes = [i32, i32, i32, i32, i32, i32, i32, i32,
                                               ctypes.POINTER(ctypes.c_size_t)]
    lib.rb_relay_sys_grid.argtypes = [i32, i32, i32, i32, i64, i32, ctypes.POINTER(i32)]
    lib.rb_relay_workspace_bytes.argtypes = [i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                             ctypes.POINTER(ctypes.c_size_t)]
    lib.rb_relay_attention.argtypes = [
        vp, i64, i64, vp, i32, i32, i32, i32, i32, i32,   # q .. d
        vp, vp, i32, i64, i64,                            # sys_k .. sys_stride_head
        vp, vp, vp, i32, i32, vp, i64, i64, i64, vp,      # k .. ctx_lens
        f32, i32, vp, i32, vp, i32, vp, ctypes.c_size_t, i32,   # scale .. phases
        vp, vp, vp, vp, vp]                               # k_new, v_new, slot_mapping, req_order, stream
    lib.rb_relay_fusion.argtypes = [vp, vp, vp, vp, vp, vp, i64, i32, vp]
    lib.rb_kv_append.argtypes = [vp, vp, vp, i32, vp, vp, i32, i32, i32, i64, i64, i64, vp]
    lib.rb_rope_rows.argtypes = [vp, vp, vp, i64, i32, ctypes.c_double, vp]
    lib.rb_rope_append.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, ctypes.c_double,
                                   vp, vp, i32, i64, i64, i64, vp]
    for name in EXPORTS:
        if name not in ("rb_last_error", "rb_abi_version"):
            getattr(lib, name).restype = i32
    if lib.rb_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI mismatch; rebuild")
    return lib


def check(status: int, what: str = "") -> None:
    if status == RB_OK:
        return
    msg = load().rb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == RB_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == RB_ERR_CONTRACT:
        raise ContractError(msg)
    raise KernelError(msg)


def sys_plan(n_rows: int, hq: int, hkv: int, s: int, grid_cap: int):
    """(fields dict, workspace bytes) of rb_system_attention's stream-K plan."""
    f = (ctypes.c_longlong * 8)()
    ws = ctypes.c_size_t(0)
    check(load().rb_sys_plan_query(n_rows, hq, hkv, s, grid_cap, f, ctypes.byref(ws)),
          "rb_sys_plan_query")
    keys = ("nq", "n_qt", "tpu", "n_units", "total", "grid", "max_parts", "rr")
    return dict(zip(keys, list(f)[:8])), ws.value


def relay_workspace_bytes(n_rows: int, hq: int, hkv: int, s: int, grid_cap: int, b: int,
                          max_rows: int, max_ctx_len: int, sm_count: int) -> int:
    out = ctypes.c_size_t(0)
    check(load().rb_relay_workspace_bytes(n_rows, hq, hkv, s, grid_cap, b, max_rows, max_ctx_len,
                                          sm_count, ctypes.byref(out)),
          "rb_relay_workspace_bytes")
    return out.value


def context_workspace_bytes(b: int, n_rows: int, max_rows: int, hq: int, hkv: int, s_prefix: int,
                            max_ctx_len: int, sm_count: int) -> int:
    out = ctypes.c_size_t(0)
    check(load().rb_context_workspace_bytes(b, n_rows, max_rows, hq, hkv, s_prefix, max_ctx_len,
                                            sm_count, ctypes.byref(out)),
          "rb_context_workspace_bytes")
    return out.value


def relay_sys_grid(n_rows: int, hq: int, hkv: int, s: int, ctx_tokens: int, sm_count: int) -> int:
    """System-kernel CTA count of the concurrent relay step (rb_relay_sys_grid)."""
    out = ctypes.c_int(0)
    check(load().rb_relay_sys_grid(n_rows, hq, hkv, s, ctx_tokens, sm_count, ctypes.byref(out)),
          "rb_relay_sys_grid")
    return out.value


def sm_count(device: int = 0) -> int:
    out = ctypes.c_int(0)
    check(load().rb_device_sm_count(device, ctypes.byref(out)), "rb_device_sm_count")
    return out.value
