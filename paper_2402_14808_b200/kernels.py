"""Segment-level launch wrappers over the C-ABI (torch tensors in, torch
tensors out, current CUDA stream).

This is the B200 replacement of the reference's kernel boundary
`relayserve.kernels` (/root/reference/pkg/src/relayserve/kernels.py:14-37):
instead of per-head matmul / softmax calls it launches one kernel per
attention segment.  There is no backend selection and no fallback.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .errors import ContractError, DimensionError

HEAD_DIM = 128
BACKEND = "cuda-sm100a"

_workspaces: dict = {}


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def sm_count(device=None) -> int:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    return _lib.sm_count(dev.index if dev.index is not None else torch.cuda.current_device())


def workspace(nbytes: int, device, stream_key: int, kind: str = "sys", layout=None) -> torch.Tensor:
    """Zero-initialised scratch, cached per (kind, device, stream).  kind
    "sys": rb_system_attention's stream-K partials + semaphores (the kernel
    leaves the semaphores zeroed, so the buffer is reusable without
    clearing); kind "relay": rb_relay_attention's unmerged partial slots;
    kind "ctx": the context split-K partials + counters.  The kernels only
    rearm their counters, so when the layout of the buffer changes (another
    problem shape: a former data region may now hold counters) it is
    zero-filled again; `layout` is the shape key of the call."""
    key = (kind, str(device), stream_key)
    ent = _workspaces.get(key)
    if ent is None or ent[0].numel() < nbytes:
        ent = (torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device), layout)
    elif ent[1] != layout:
        ent[0].zero_()
        ent = (ent[0], layout)
    _workspaces[key] = ent
    return ent[0]


def _check_bf16(name, t, host_ok=False):
    """bf16 with a contiguous head dim, on the GPU -- or, where `host_ok`
    (the step's inputs / output of the zero-copy e2e path), in pinned host
    memory, which the kernels address directly (UVA)."""
    on_dev = t.is_cuda or (host_ok and t.device.type == "cpu" and t.is_pinned())
    if t.dtype != torch.bfloat16 or not on_dev:
        where = "CUDA or pinned host" if host_ok else "CUDA"
        raise ContractError(f"{name}: expected a {where} bfloat16 tensor, got {t.dtype} on {t.device}")
    if t.stride(-1) != 1:
        raise ContractError(f"{name}: head_dim must be the contiguous dimension")


def _check_index(name, t, device):
    if t.dtype not in (torch.int32, torch.int64) or t.device != device or not t.is_contiguous():
        raise ContractError(f"{name}: expected a contiguous integer tensor on {device}, "
                            f"got {t.dtype} on {t.device}")
    want = torch.int64 if name == "req_offset" else torch.int32
    if t.dtype != want:
        raise ContractError(f"{name}: expected {want}, got {t.dtype}")


def system_attention(q, sys_k, sys_v, *, kv_layout="shd", scale=None, grid=None,
                     o_sys=None, lse_sys=None, ws=None):
    """Unmasked attention of every query row over the shared prefix.

    q: (n_rows, hq, 128) bf16; sys_k/sys_v: (s, hkv, 128) for kv_layout
    'shd' (the reference's layout) or (hkv, s, 128) for 'hsd' (the
    SystemKvCache layout).  Returns (o_sys fp32 (n_rows, hq, 128),
    lse_sys fp32 (n_rows, hq)), natural-log LSE.
    """
    _check_bf16("q", q)
    _check_bf16("sys_k", sys_k)
    _check_bf16("sys_v", sys_v)
    if sys_k.shape != sys_v.shape or sys_k.stride() != sys_v.stride():
        raise DimensionError(f"sys_k/sys_v shapes differ: {tuple(sys_k.shape)} vs {tuple(sys_v.shape)}")
    n_rows, hq, d = q.shape
    if kv_layout == "shd":
        s, hkv, dk = sys_k.shape
        st_tok, st_head = sys_k.stride(0), sys_k.stride(1)
    elif kv_layout == "hsd":
        hkv, s, dk = sys_k.shape
        st_tok, st_head = sys_k.stride(1), sys_k.stride(0)
    else:
        raise ContractError(f"unknown kv_layout {kv_layout!r}")
    if d != HEAD_DIM or dk != HEAD_DIM:
        raise DimensionError(f"head_dim must be {HEAD_DIM} (pad smaller dims), got {d}/{dk}")
    if hkv < 1 or hq % hkv != 0:
        raise DimensionError(f"query heads {hq} not a multiple of kv heads {hkv}")
    dev = q.device
    if o_sys is None:
        o_sys = torch.empty((n_rows, hq, HEAD_DIM), dtype=torch.float32, device=dev)
    if lse_sys is None:
        lse_sys = torch.empty((n_rows, hq), dtype=torch.float32, device=dev)
    grid = sm_count(dev) if grid is None else grid
    stream = _stream(dev)
    if ws is None:
        _, need = _lib.sys_plan(n_rows, hq, hkv, s, grid)
        ws = workspace(need, dev, stream, layout=(n_rows, hq, hkv, s, grid))
    scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else scale
    _lib.check(_lib.load().rb_system_attention(
        q.data_ptr(), q.stride(0), q.stride(1), n_rows, hq, hkv, HEAD_DIM,
        sys_k.data_ptr(), sys_v.data_ptr(), s, st_tok, st_head, float(scale), grid,
        o_sys.data_ptr(), lse_sys.data_ptr(), ws.data_ptr(), ws.numel(), stream),
        "rb_system_attention")
    return o_sys, lse_sys


def context_attention(q, q_start, k, v, ctx_lens, *, max_rows, hkv,
                      block_table=None, block_size=0, req_offset=None,
                      strides=None, causal=True, prefix_k=None, prefix_v=None,
                      prefix_strides=None, o_sys=None, lse_sys=None, scale=None,
                      out=None, out_fp32=False, lse_out=None, want_lse=True,
                      max_ctx_len=0, ws=None):
    """Context (or relay, or naive-baseline) attention; see
    include/relay_b200.h:rb_context_attention for the addressing modes.

    q: (n_rows, hq, 128) bf16; q_start int32 (b+1,); ctx_lens int32 (b,).
    strides = (stride_block, stride_tok, stride_head) in elements.
    max_ctx_len: an upper bound of ctx_lens (0: unknown) -- enables the
    split-K over long contexts; its workspace is cached per stream unless
    `ws` (zero-filled, rb_context_workspace_bytes) is given.
    """
    _check_bf16("q", q)
    _check_bf16("k", k)
    _check_bf16("v", v)
    _check_index("q_start", q_start, q.device)
    _check_index("ctx_lens", ctx_lens, q.device)
    for name, t in (("block_table", block_table), ("req_offset", req_offset)):
        if t is not None:
            _check_index(name, t, q.device)
    if prefix_k is not None:
        _check_bf16("prefix_k", prefix_k)
        _check_bf16("prefix_v", prefix_v)
    n_rows, hq, d = q.shape
    if d != HEAD_DIM:
        raise DimensionError(f"head_dim must be {HEAD_DIM}, got {d}")
    b = ctx_lens.numel()
    if q_start.numel() != b + 1:
        raise DimensionError(f"q_start needs b + 1 = {b + 1} offsets, got {q_start.numel()}")
    dev = q.device
    if out is None:
        out = torch.empty((n_rows, hq, HEAD_DIM),
                          dtype=torch.float32 if out_fp32 else torch.bfloat16, device=dev)
    out_fp32 = out.dtype == torch.float32
    if lse_out is None and want_lse:
        lse_out = torch.empty((n_rows, hq), dtype=torch.float32, device=dev)
    s_prefix = 0
    p_tok = p_head = 0
    if prefix_k is not None:
        s_prefix = prefix_strides[2]
        p_tok, p_head = prefix_strides[0], prefix_strides[1]
    sb, stok, sh = strides
    bt_stride = block_table.stride(0) if block_table is not None else 0
    scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else scale
    stream = _stream(dev)
    if ws is None and max_ctx_len > 0:
        need = _lib.context_workspace_bytes(b, n_rows, max_rows, hq, hkv, s_prefix, max_ctx_len,
                                            sm_count(dev))
        ws = workspace(need, dev, stream, kind="ctx",
                       layout=(b, n_rows, max_rows, hq, hkv, s_prefix, max_ctx_len)) if need else None
    _lib.check(_lib.load().rb_context_attention(
        q.data_ptr(), q.stride(0), q.stride(1), q_start.data_ptr(), b, n_rows, max_rows, hq, hkv,
        HEAD_DIM, k.data_ptr(), v.data_ptr(), _ptr(block_table), bt_stride, block_size,
        _ptr(req_offset), sb, stok, sh, ctx_lens.data_ptr(), 1 if causal else 0,
        _ptr(prefix_k), _ptr(prefix_v), s_prefix, p_tok, p_head, _ptr(o_sys), _ptr(lse_sys),
        float(scale), out.data_ptr(), 1 if out_fp32 else 0, _ptr(lse_out), int(max_ctx_len),
        _ptr(ws), 0 if ws is None else ws.numel(), stream),
        "rb_context_attention")
    return out, lse_out


def relay_attention(q, q_start, sys_k, sys_v, k, v, ctx_lens, *, max_rows, hkv,
                    sys_layout="hsd", block_table=None, block_size=0, req_offset=None,
                    strides=None, scale=None, grid=None, out=None, lse_out=None,
                    out_fp32=False, ws=None, phases=3, max_ctx_len=0, k_new=None, v_new=None,
                    slot_mapping=None, req_order=None):
    """The fused relay step (rb_relay_attention): system kernel (stream-K
    partials, no merge) + context kernel whose epilogue merges the system
    partials with the context state.  Returns (out, lse).  max_ctx_len: an
    upper bound of ctx_lens (0: unknown) for the context split-K; `ws` must
    then hold rb_relay_workspace_bytes(..., max_ctx_len, sm_count) bytes.
    k_new / v_new (n_rows, hkv, 128) bf16 + slot_mapping int32 (n_rows,):
    the fused append of the step's new tokens (paged layout; the tensors may
    be pinned host memory); ctx_lens must already count them.  req_order
    (int32 (b,), a permutation of the requests, optional): the order the
    context kernel claims their work in (longest context first balances
    varied lengths); the results do not depend on it."""
    # q (and out) may live in pinned host memory (zero-copy e2e step); the
    # caches, indices and workspace are on the device
    _check_bf16("q", q, host_ok=True)
    for name, t in (("sys_k", sys_k), ("sys_v", sys_v), ("k", k), ("v", v)):
        _check_bf16(name, t)
        if t.device != sys_k.device:
            raise ContractError(f"{name} is on {t.device}, sys_k on {sys_k.device}")
    _check_index("q_start", q_start, sys_k.device)
    _check_index("ctx_lens", ctx_lens, sys_k.device)
    for name, t in (("block_table", block_table), ("req_offset", req_offset)):
        if t is not None:
            _check_index(name, t, sys_k.device)
    n_rows, hq, d = q.shape
    if d != HEAD_DIM:
        raise DimensionError(f"head_dim must be {HEAD_DIM}, got {d}")
    if q_start.numel() != ctx_lens.numel() + 1:
        raise DimensionError(f"q_start needs b + 1 = {ctx_lens.numel() + 1} offsets, "
                             f"got {q_start.numel()}")
    if (k_new is None) != (v_new is None) or (k_new is None) != (slot_mapping is None):
        raise ContractError("k_new, v_new and slot_mapping go together")
    if k_new is not None:
        for name, t in (("k_new", k_new), ("v_new", v_new)):
            _check_bf16(name, t, host_ok=True)
            if not t.is_contiguous() or tuple(t.shape) != (q.shape[0], hkv, HEAD_DIM):
                raise DimensionError(f"{name} must be contiguous ({q.shape[0]}, {hkv}, {HEAD_DIM})")
        _check_index("slot_mapping", slot_mapping, sys_k.device)
    if req_order is not None:
        _check_index("req_order", req_order, sys_k.device)
        if req_order.numel() != ctx_lens.numel():
            raise DimensionError(f"req_order needs b = {ctx_lens.numel()} entries, got {req_order.numel()}")
    for name, t in (("out", out), ("lse_out", lse_out)):
        if t is not None and not (t.is_cuda or (t.device.type == "cpu" and t.is_pinned())):
            raise ContractError(f"{name}: expected a CUDA or pinned host tensor")
    if sys_k.shape != sys_v.shape or k.shape != v.shape:
        raise DimensionError("K and V shapes differ")
    if sys_layout == "hsd":
        _, s, _ = sys_k.shape
        s_tok, s_head = sys_k.stride(1), sys_k.stride(0)
    else:
        s, _, _ = sys_k.shape
        s_tok, s_head = sys_k.stride(0), sys_k.stride(1)
    dev = sys_k.device
    b = ctx_lens.numel()
    if out is None:
        out = torch.empty((n_rows, hq, HEAD_DIM),
                          dtype=torch.float32 if out_fp32 else torch.bfloat16, device=dev)
    if lse_out is None:
        lse_out = torch.empty((n_rows, hq), dtype=torch.float32, device=dev)
    grid = sm_count(dev) if grid is None else grid
    stream = _stream(dev)
    if ws is None:
        need = _lib.relay_workspace_bytes(n_rows, hq, hkv, s, grid, b, max_rows, max_ctx_len,
                                          sm_count(dev))
        ws = workspace(need, dev, stream, kind="relay",
                       layout=(n_rows, hq, hkv, s, grid, b, max_rows, max_ctx_len))
    sb, stok, sh = strides
    bt_stride = block_table.stride(0) if block_table is not None else 0
    scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else scale
    _lib.check(_lib.load().rb_relay_attention(
        q.data_ptr(), q.stride(0), q.stride(1), q_start.data_ptr(), b, n_rows, max_rows, hq, hkv,
        HEAD_DIM, sys_k.data_ptr(), sys_v.data_ptr(), s, s_tok, s_head, k.data_ptr(),
        v.data_ptr(), _ptr(block_table), bt_stride, block_size, _ptr(req_offset), sb, stok, sh,
        ctx_lens.data_ptr(), float(scale), grid, out.data_ptr(),
        1 if out.dtype == torch.float32 else 0, lse_out.data_ptr(), int(max_ctx_len),
        ws.data_ptr(), ws.numel(), phases, _ptr(k_new), _ptr(v_new), _ptr(slot_mapping),
        _ptr(req_order), stream),
        "rb_relay_attention")
    return out, lse_out


def relay_fusion_fp32(o_sys, lse_sys, o_ctx, lse_ctx, out=None, lse_out=None):
    """Standalone fusion kernel on fp32 CUDA tensors of matching shapes."""
    tens = [o_sys, lse_sys, o_ctx, lse_ctx]
    if any((not t.is_cuda) or t.dtype != torch.float32 or not t.is_contiguous() for t in tens):
        raise ContractError("relay_fusion_fp32 expects contiguous fp32 CUDA tensors")
    d = o_sys.shape[-1]
    n_vec = lse_sys.numel()
    out = torch.empty_like(o_sys) if out is None else out
    lse_out = torch.empty_like(lse_sys) if lse_out is None else lse_out
    _lib.check(_lib.load().rb_relay_fusion(
        o_sys.data_ptr(), lse_sys.data_ptr(), o_ctx.data_ptr(), lse_ctx.data_ptr(),
        out.data_ptr(), lse_out.data_ptr(), n_vec, d, _stream(o_sys.device)), "rb_relay_fusion")
    return out, lse_out


def kv_append(k_new, v_new, slot_mapping, k_pool, v_pool, block_size):
    """Scatter (n_tok, hkv, 128) new rows into a [num_blocks][hkv][bs][128] pool.
    k_new / v_new may be pinned host tensors (read directly by the kernel)."""
    _check_bf16("k_new", k_new, host_ok=True)
    _check_bf16("v_new", v_new, host_ok=True)
    n_tok, hkv, d = k_new.shape
    _lib.check(_lib.load().rb_kv_append(
        k_new.data_ptr(), v_new.data_ptr(), slot_mapping.data_ptr(), n_tok, k_pool.data_ptr(),
        v_pool.data_ptr(), hkv, d, block_size, k_pool.stride(0), k_pool.stride(2),
        k_pool.stride(1), _stream(k_pool.device)), "rb_kv_append")


ROPE_BASE = 10000.0  # numerics.ROPE_BASE / model.py:292


def rope_rows(x, positions, base=ROPE_BASE, out=None):
    """`kernels.rope_rows` (_kernels_cy.pyx:80-102) on the GPU: row i's
    consecutive pairs rotated by positions[i] * base^(-2j/d).  x: fp32 CUDA
    (n, d), d even; positions: int64 (n,); angles and rotation in fp64."""
    if x.dim() != 2 or x.shape[1] % 2 != 0:
        raise DimensionError(f"rope_rows requires (n, even d) rows, got {tuple(x.shape)}")
    if x.dtype != torch.float32 or not x.is_contiguous():
        raise ContractError("rope_rows takes contiguous fp32 rows")
    positions = positions.to(device=x.device, dtype=torch.int64).contiguous()
    if positions.shape != (x.shape[0],):
        raise DimensionError("rope_rows: positions must be one per row")
    out = torch.empty_like(x) if out is None else out
    _lib.check(_lib.load().rb_rope_rows(x.data_ptr(), out.data_ptr(), positions.data_ptr(),
                                        x.shape[0], x.shape[1], float(base),
                                        _stream(x.device)), "rb_rope_rows")
    return out


def rope_append(q, k_new, v_new, positions, slot_mapping, k_pool, v_pool, block_size,
                base=ROPE_BASE, q_out=None):
    """Decode-step prologue in one launch: q (n_tok, hq, 128) and k_new
    (n_tok, hkv, 128) rotated to `positions` (int64, one per token), the
    rotated K and raw V scattered into a [num_blocks][hkv][bs][128] pool at
    `slot_mapping` (int32).  Returns the rotated q (in place if q_out is q)."""
    for name, t in (("q", q), ("k_new", k_new), ("v_new", v_new)):
        _check_bf16(name, t)
    n_tok, hq, d = q.shape
    hkv = k_new.shape[1]
    if k_new.shape != v_new.shape or k_new.shape[0] != n_tok:
        raise DimensionError(f"rope_append: k/v {tuple(k_new.shape)} vs q {tuple(q.shape)}")
    q_out = torch.empty_like(q) if q_out is None else q_out
    positions = positions.to(device=q.device, dtype=torch.int64).contiguous()
    _lib.check(_lib.load().rb_rope_append(
        q.data_ptr(), q_out.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), positions.data_ptr(),
        slot_mapping.data_ptr(), n_tok, hq, hkv, d, float(base), k_pool.data_ptr(),
        v_pool.data_ptr(), block_size, k_pool.stride(0), k_pool.stride(2), k_pool.stride(1),
        _stream(q.device)), "rb_rope_append")
    return q_out


def umma_probe(k, q, v, p):
    """Debug: run the system kernel's tcgen05 operand layouts on one tile."""
    nq = q.shape[0]
    s_out = torch.empty((128, nq), dtype=torch.float32, device=k.device)
    o_out = torch.empty((128, nq), dtype=torch.float32, device=k.device)
    _lib.check(_lib.load_diag().rb_debug_umma_probe(
        k.data_ptr(), q.data_ptr(), v.data_ptr(), p.data_ptr(), nq, s_out.data_ptr(),
        o_out.data_ptr(), _stream(k.device)), "rb_debug_umma_probe")
    return s_out, o_out
