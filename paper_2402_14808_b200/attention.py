"""RelayAttention operator API on B200 -- a drop-in for the reference's
`relayserve.attention` hot path (/root/reference/pkg/src/relayserve/attention.py).

Same names, argument meaning and error behaviour as the reference:

  TrafficCounter, LseAttentionOutput          attention.py:28-69
  naive_causal_attention(q, k, v)             attention.py:72-93
  attention_with_lse(q, k, v, causal)         attention.py:96-134
  relay_fusion(o_sys, lse_sys, o_ctx, lse_ctx)  attention.py:137-157
  relay_attention_ragged(...)                 attention.py:203-243
  relay_attention(...)                        attention.py:246-263
  baseline_attention_ragged / baseline_attention  attention.py:266-296

Inputs may be numpy arrays (the reference's float64 convention; results
come back as float64 numpy) or torch tensors (results stay on the GPU, fp32).
Either way the arithmetic runs in the sm_100a kernels of librelay_b200.so:
bf16 operands, fp32 accumulation and softmax, natural-log LSE.  Extensions
over the reference: GQA (query heads a multiple of KV heads; the reference
raises DimensionError, attention.py:109-110), and `return_lse` on the relay
entry points (the fused LSE = logaddexp(lse_sys, lse_ctx)).

Paged-native fast path for serving / benchmarking: RelayDecodeStep and
NaiveDecodeStep run one decode step over a SystemKvCache + PagedKvCache
with preallocated buffers (CUDA-graph capturable).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .errors import ContractError, DimensionError

HEAD_DIM = kernels.HEAD_DIM


@dataclass
class TrafficCounter:
    """Per-step element-access accounting (attention.py:28-57): one attended
    position costs h*d elements for its K/V pair; LSE scalars are separate."""

    elements_read: int = 0
    elements_written: int = 0
    lse_elements: int = 0

    def add_load(self, n: int):
        self.elements_read += n

    def add_store(self, n: int):
        self.elements_read += n
        self.elements_written += n

    def add_lse(self, n: int):
        self.lse_elements += n

    def reset(self):
        self.elements_read = 0
        self.elements_written = 0
        self.lse_elements = 0


@dataclass
class LseAttentionOutput:
    """output (b, m, h, d) and lse (b, m, h)."""

    output: object
    lse: object


# ----------------------------------------------------------------- helpers

def _is_numpy(x):
    return isinstance(x, np.ndarray) or not isinstance(x, torch.Tensor)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else tuple(np.shape(x))


def _ndim(x, nd, name):
    if len(_shape(x)) != nd:
        raise DimensionError(f"{name}: expected {nd} dimensions, got {len(_shape(x))}")


def _to_dev_bf16(x, device):
    """Any array -> CUDA bf16, head_dim zero-padded to 128 (exact)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device)
    d = t.shape[-1]
    if d > HEAD_DIM:
        raise DimensionError(f"head_dim {d} > {HEAD_DIM} is not supported")
    t = t.to(torch.bfloat16)
    if d < HEAD_DIM:
        t = torch.nn.functional.pad(t, (0, HEAD_DIM - d))
    return t.contiguous()


def _out(t, d, like_numpy):
    t = t[..., :d] if t.shape[-1] != d else t
    if like_numpy:
        return t.detach().to("cpu", torch.float64).numpy()
    return t


def _lse_out(t, like_numpy):
    if like_numpy:
        return t.detach().to("cpu", torch.float64).numpy()
    return t


# ------------------------------------------------------------------- ops

def attention_with_lse(q, k, v, causal):
    """Scaled dot-product attention with per-query natural-log LSE.

    q: (b, m, h, d); k, v: (b, n, h_kv, d).  causal=True: query t attends
    keys 0..(n - m + t) (attention.py:120-121); causal=False: all n keys.
    b == 1 and not causal (the shared-prefix case, attention.py:184-185)
    runs the tcgen05 system kernel; everything else the context kernel.
    """
    _ndim(q, 4, "q")
    _ndim(k, 4, "k")
    _ndim(v, 4, "v")
    qs, ks = _shape(q), _shape(k)
    b, m, h, d = qs
    if ks != _shape(v):
        raise DimensionError(f"k/v shapes differ: {ks} vs {_shape(v)}")
    if ks[0] != b or ks[3] != d or ks[2] < 1 or h % ks[2] != 0:
        raise DimensionError(f"k {ks} incompatible with q {qs}")
    n, hkv = ks[1], ks[2]
    if n < 1:
        raise ContractError("attention requires at least one key")
    if causal and n < m:
        raise ContractError(f"causal attention needs n >= m, got n={n}, m={m}")
    like_np = _is_numpy(q)
    dev = q.device if isinstance(q, torch.Tensor) else _device()
    scale = 1.0 / math.sqrt(d)
    qd = _to_dev_bf16(q, dev).reshape(b * m, h, HEAD_DIM)
    kd = _to_dev_bf16(k, dev)
    vd = _to_dev_bf16(v, dev)
    if b == 1 and not causal:
        o, lse = kernels.system_attention(qd, kd[0], vd[0], kv_layout="shd", scale=scale)
    else:
        q_start = torch.arange(0, b * m + 1, m, dtype=torch.int32, device=dev)
        req_off = torch.arange(0, b * n, n, dtype=torch.int64, device=dev)
        lens = torch.full((b,), n, dtype=torch.int32, device=dev)
        kf = kd.reshape(b * n, hkv, HEAD_DIM)
        vf = vd.reshape(b * n, hkv, HEAD_DIM)
        o, lse = kernels.context_attention(
            qd, q_start, kf, vf, lens, max_rows=m * (h // hkv), hkv=hkv, req_offset=req_off,
            strides=(0, kf.stride(0), kf.stride(1)), causal=causal, scale=scale, out_fp32=True,
            max_ctx_len=n)
    return LseAttentionOutput(output=_out(o.reshape(b, m, h, HEAD_DIM), d, like_np),
                              lse=_lse_out(lse.reshape(b, m, h), like_np))


def naive_causal_attention(q, k, v):
    """Brute-force-equivalent causal self-attention over one sequence
    (attention.py:72-93): q, k, v (l, h, d); position t attends 0..t."""
    _ndim(q, 3, "q")
    _ndim(k, 3, "k")
    _ndim(v, 3, "v")
    if not (_shape(q) == _shape(k) == _shape(v)):
        raise DimensionError(f"q/k/v shapes differ: {_shape(q)}, {_shape(k)}, {_shape(v)}")
    res = attention_with_lse(q[None], k[None], v[None], causal=True)
    return res.output[0]


def relay_fusion(o_sys, lse_sys, o_ctx, lse_ctx):
    """alpha_sys = 1/(1+exp(lse_ctx - lse_sys)); o = alpha*o_sys + (1-alpha)*o_ctx
    (attention.py:137-157), on the GPU in fp32 with max-subtracted weights."""
    _ndim(o_sys, 4, "o_sys")
    _ndim(o_ctx, 4, "o_ctx")
    _ndim(lse_sys, 3, "lse_sys")
    _ndim(lse_ctx, 3, "lse_ctx")
    if _shape(o_sys) != _shape(o_ctx):
        raise DimensionError(f"output shapes differ: {_shape(o_sys)} vs {_shape(o_ctx)}")
    if _shape(lse_sys) != _shape(lse_ctx) or _shape(lse_sys) != _shape(o_sys)[:3]:
        raise DimensionError("lse shapes must match output batch/query/head dims")
    like_np = _is_numpy(o_sys)
    dev = o_sys.device if isinstance(o_sys, torch.Tensor) else _device()

    def f32(x):
        if isinstance(x, torch.Tensor):
            return x.to(device=dev, dtype=torch.float32).contiguous()
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)

    out, _ = kernels.relay_fusion_fp32(f32(o_sys), f32(lse_sys), f32(o_ctx), f32(lse_ctx))
    return out.to("cpu", torch.float64).numpy() if like_np else out


def _count_relay(counter, m_list, c_list, s, h, d):
    """TrafficCounter updates of attention.py:168-173, 186-192, 238-242."""
    hd = h * d
    for m, c in zip(m_list, c_list):
        counter.add_load(m * hd)
        counter.add_load(c * hd)
        counter.add_store(m * hd)
        counter.add_lse(m * h)
    total_m = sum(m_list)
    counter.add_load(total_m * hd)
    counter.add_load(s * hd)
    counter.add_store(total_m * hd)
    counter.add_lse(total_m * h)
    for m in m_list:
        counter.add_load(2 * m * h * d)
        counter.add_store(m * h * d)
        counter.add_lse(2 * m * h)


def relay_attention_ragged(q_list, sys_k, sys_v, ctx_k, ctx_v, counter=None,
                           system_first=False, return_lse=False):
    """Relay attention for requests with different query counts
    (attention.py:203-243).  q_list[r]: (m_r, h, d); ctx_k[r]/ctx_v[r]:
    (c_r, h_kv, d) including the current tokens; sys_k/sys_v: (s, h_kv, d),
    s >= 1.  Equals causal attention over [system || context] per request.

    One rb_relay_attention call: the system segment runs once for the whole
    batch (tcgen05 kernel), the context segment and the fusion run in one
    kernel.  Fusion is a
    single deterministic LSE merge, so `system_first` cannot change the
    result (the reference's bitwise order-independence, attention.py:208-212).
    """
    _ndim(sys_k, 3, "sys_k")
    _ndim(sys_v, 3, "sys_v")
    if _shape(sys_k) != _shape(sys_v):
        raise DimensionError(f"sys_k/sys_v shapes differ: {_shape(sys_k)} vs {_shape(sys_v)}")
    if _shape(sys_k)[0] < 1:
        raise ContractError("relay attention requires a non-empty system segment; "
                            "use the baseline path when there is no shared prefix")
    if not (len(q_list) == len(ctx_k) == len(ctx_v)):
        raise DimensionError("one context k/v pair required per request")
    for qr in q_list:
        _ndim(qr, 3, "q")
    for kr in list(ctx_k) + list(ctx_v):
        _ndim(kr, 3, "ctx_k")
    s, hkv, d = _shape(sys_k)
    b = len(q_list)
    m_list = [_shape(qr)[0] for qr in q_list]
    c_list = [_shape(kr)[0] for kr in ctx_k]
    h = _shape(q_list[0])[1] if b else hkv
    for qr, kr, vr in zip(q_list, ctx_k, ctx_v):
        if _shape(qr)[1:] != (h, d) or _shape(kr)[1:] != (hkv, d) or _shape(kr) != _shape(vr):
            raise DimensionError("q/context shapes inconsistent with the system cache")
    if hkv < 1 or h % hkv != 0:
        raise DimensionError(f"query heads {h} not a multiple of kv heads {hkv}")
    for m, c in zip(m_list, c_list):
        if c < m:
            raise ContractError(f"causal attention needs n >= m, got n={c}, m={m}")
    if b == 0:
        return ([], []) if return_lse else []
    like_np = _is_numpy(q_list[0])
    dev = q_list[0].device if isinstance(q_list[0], torch.Tensor) else _device()
    scale = 1.0 / math.sqrt(d)

    def cat(lst):
        if isinstance(lst[0], torch.Tensor):
            return torch.cat([x.to(dev) for x in lst], 0)
        return np.concatenate([np.asarray(x) for x in lst], 0)

    qf = _to_dev_bf16(cat(q_list), dev)
    skd = _to_dev_bf16(sys_k, dev)
    svd = _to_dev_bf16(sys_v, dev)
    ckd = _to_dev_bf16(cat(list(ctx_k)), dev)
    cvd = _to_dev_bf16(cat(list(ctx_v)), dev)
    q_start = torch.tensor(np.concatenate([[0], np.cumsum(m_list)]), dtype=torch.int32, device=dev)
    req_off = torch.tensor(np.concatenate([[0], np.cumsum(c_list)[:-1]]), dtype=torch.int64,
                           device=dev)
    lens = torch.tensor(c_list, dtype=torch.int32, device=dev)

    out, lse = kernels.relay_attention(
        qf, q_start, skd, svd, ckd, cvd, lens, max_rows=max(m_list) * (h // hkv), hkv=hkv,
        sys_layout="shd", req_offset=req_off, strides=(0, ckd.stride(0), ckd.stride(1)),
        scale=scale, out_fp32=True, max_ctx_len=max(c_list))
    if counter is not None:
        _count_relay(counter, m_list, c_list, s, h, d)
    outs, lses, row = [], [], 0
    for m in m_list:
        outs.append(_out(out[row:row + m], d, like_np))
        lses.append(_lse_out(lse[row:row + m], like_np))
        row += m
    return (outs, lses) if return_lse else outs


def relay_attention(q, sys_k, sys_v, ctx_k, ctx_v, counter=None, system_first=False,
                    return_lse=False):
    """Uniform-batch relay attention (attention.py:246-263).
    q: (b, m, h, d); ctx_k[r]/ctx_v[r]: (c_r, h_kv, d)."""
    _ndim(q, 4, "q")
    b = _shape(q)[0]
    if len(ctx_k) != b or len(ctx_v) != b:
        raise DimensionError(f"expected {b} context caches, got {len(ctx_k)}/{len(ctx_v)}")
    res = relay_attention_ragged([q[r] for r in range(b)], sys_k, sys_v, ctx_k, ctx_v,
                                 counter=counter, system_first=system_first,
                                 return_lse=return_lse)
    stack = (lambda xs: np.stack(xs, 0)) if _is_numpy(q) else (lambda xs: torch.stack(xs, 0))
    if return_lse:
        return stack(res[0]), stack(res[1])
    return stack(res)


def baseline_attention_ragged(q_list, full_k, full_v, counter=None):
    """Per-request causal attention over each request's full cache
    (attention.py:266-288) -- the shared prefix replicated per request."""
    if not (len(q_list) == len(full_k) == len(full_v)):
        raise DimensionError("one k/v pair required per request")
    outs = []
    for qr, kr, vr in zip(q_list, full_k, full_v):
        _ndim(qr, 3, "q")
        _ndim(kr, 3, "k")
        _ndim(vr, 3, "v")
    b = len(q_list)
    if b == 0:
        return outs
    m_list = [_shape(x)[0] for x in q_list]
    n_list = [_shape(x)[0] for x in full_k]
    h, d = _shape(q_list[0])[1:]
    hkv = _shape(full_k[0])[1]
    for m, n in zip(m_list, n_list):
        if n < 1:
            raise ContractError("attention requires at least one key")
        if n < m:
            raise ContractError(f"causal attention needs n >= m, got n={n}, m={m}")
    like_np = _is_numpy(q_list[0])
    dev = q_list[0].device if isinstance(q_list[0], torch.Tensor) else _device()

    def cat(lst):
        if isinstance(lst[0], torch.Tensor):
            return torch.cat([x.to(dev) for x in lst], 0)
        return np.concatenate([np.asarray(x) for x in lst], 0)

    qf = _to_dev_bf16(cat(q_list), dev)
    kd = _to_dev_bf16(cat(list(full_k)), dev)
    vd = _to_dev_bf16(cat(list(full_v)), dev)
    q_start = torch.tensor(np.concatenate([[0], np.cumsum(m_list)]), dtype=torch.int32, device=dev)
    req_off = torch.tensor(np.concatenate([[0], np.cumsum(n_list)[:-1]]), dtype=torch.int64,
                           device=dev)
    lens = torch.tensor(n_list, dtype=torch.int32, device=dev)
    out, _ = kernels.context_attention(
        qf, q_start, kd, vd, lens, max_rows=max(m_list) * (h // hkv), hkv=hkv, req_offset=req_off,
        strides=(0, kd.stride(0), kd.stride(1)), causal=True, scale=1.0 / math.sqrt(d),
        out_fp32=True, want_lse=False, max_ctx_len=max(n_list))
    if counter is not None:
        for m, n in zip(m_list, n_list):
            hd = h * d
            counter.add_load(m * hd)
            counter.add_load(n * hd)
            counter.add_store(m * hd)
    row = 0
    for m in m_list:
        outs.append(_out(out[row:row + m], d, like_np))
        row += m
    return outs


def baseline_attention(q, full_k, full_v, counter=None):
    """Uniform-batch baseline (attention.py:291-296)."""
    _ndim(q, 4, "q")
    outs = baseline_attention_ragged([q[r] for r in range(_shape(q)[0])], full_k, full_v,
                                     counter=counter)
    return np.stack(outs, 0) if _is_numpy(q) else torch.stack(outs, 0)


# ------------------------------------------------------ paged decode steps

class RelayDecodeStep:
    """One relay decode step (m = 1 token per request) over resident caches.

    q: (b, hq, 128) bf16 -> out (b, hq, 128) bf16 and fused lse (b, hq) fp32.
    One rb_relay_attention call = two kernels on the current stream: the
    tcgen05 system kernel (shared prefix read once, stream-K partials left
    unmerged, each unit published on a counter) on a byte-proportional share
    of the SMs, and the paged context kernel, launched with programmatic
    dependent launch so it streams concurrently on the other SMs, whose
    epilogue merges the system partials with the context state (relay
    fusion).  All buffers are preallocated, so the step
    can be captured in a CUDA graph.
    """

    def __init__(self, sys_cache, paged_cache, block_table, ctx_lens, hq, layer=0,
                 grid=None, out_dtype=torch.bfloat16, scale=None, out=None, lse=None):
        self.sys_cache, self.paged, self.layer = sys_cache, paged_cache, layer
        self.block_table = block_table
        self.ctx_lens = ctx_lens
        self.b = ctx_lens.numel()
        self.hq = hq
        self.hkv = sys_cache.kv_heads
        if hq % self.hkv != 0 or paged_cache.kv_heads != self.hkv:
            raise DimensionError("query heads must be a multiple of the (shared) kv heads")
        if block_table.dim() != 2 or block_table.shape[0] != self.b:
            raise DimensionError(f"block_table must be (b={self.b}, max_blocks), "
                                 f"got {tuple(block_table.shape)}")
        for name, t in (("block_table", block_table), ("ctx_lens", ctx_lens)):
            if t.dtype != torch.int32 or not t.is_cuda:
                raise ContractError(f"{name}: expected a CUDA int32 tensor, got {t.dtype} on {t.device}")
        for t in (sys_cache.keys[layer], sys_cache.values[layer], paged_cache.k_pool):
            if not t.is_cuda or t.device != block_table.device:
                raise ContractError("caches, block table and context lengths must share one CUDA device")
        # softmax temperature of the model's head dim (a d=16 cache is zero-
        # padded to 128 on the device; the scale stays 16 ** -0.5)
        self.scale = sys_cache.scale if scale is None else float(scale)
        dev = block_table.device
        from . import _lib
        if grid is None:
            # concurrent split: system CTAs by their share of the step's HBM bytes
            grid = _lib.relay_sys_grid(self.b, hq, self.hkv, sys_cache.system_len,
                                       int(ctx_lens.sum().item()), kernels.sm_count(dev))
        # the block table's capacity bounds every context it can address, so
        # the split-K plan stays valid while the contexts grow into it
        self.max_ctx_len = block_table.shape[1] * paged_cache.block_size
        self.ws = None
        self._set_grid(grid)
        self.out = torch.empty((self.b, hq, HEAD_DIM), dtype=out_dtype, device=dev) if out is None else out
        self.lse = torch.empty((self.b, hq), dtype=torch.float32, device=dev) if lse is None else lse
        if tuple(self.out.shape) != (self.b, hq, HEAD_DIM) or tuple(self.lse.shape) != (self.b, hq):
            raise DimensionError("out / lse buffers must be (b, hq, 128) / (b, hq)")
        self.q_start = torch.arange(self.b + 1, dtype=torch.int32, device=dev)
        # a system-only launch (profiling) leaves its units published; the
        # next full step must start from rearmed counters
        self._system_pending = False
        # claim order of the requests' context work: longest first when the
        # lengths differ (each context CTA claims a few items ahead, and a long
        # item queued at the end of the pool is a tail); None when uniform
        self.req_order = None
        if self.b > 1 and int(ctx_lens.max().item()) != int(ctx_lens.min().item()):
            self.req_order = torch.empty(self.b, dtype=torch.int32, device=dev)
            self.reorder()

    def reorder(self):
        """Recompute the context claim order from the current ctx_lens (in
        place, so a captured CUDA graph keeps using it; device-side, no sync).
        Results never depend on the order."""
        if self.req_order is not None:
            self.req_order.copy_(torch.argsort(self.ctx_lens, descending=True, stable=True))

    def _set_grid(self, grid):
        from . import _lib
        if grid < 1:
            raise ContractError(f"grid must be >= 1 system CTAs, got {grid}")
        dev = self.block_table.device
        self.grid = grid
        self.plan, _ = _lib.sys_plan(self.b, self.hq, self.hkv, self.sys_cache.system_len, grid)
        need = max(256, _lib.relay_workspace_bytes(self.b, self.hq, self.hkv,
                                                   self.sys_cache.system_len, grid, self.b,
                                                   self.hq // self.hkv, self.max_ctx_len,
                                                   kernels.sm_count(dev)))
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.zeros(need, dtype=torch.uint8, device=dev)
        else:
            self.ws.zero_()   # the counters / partial layout follow the plan
        self._system_pending = False

    def resplit(self, ctx_tokens):
        """Recompute the SM split of the two kernels for the batch's current
        total context length (the split set at construction goes stale as a
        serving loop's contexts grow; the host knows the lengths, so no
        device read is needed).  Returns True when the split changed (a CUDA
        graph captured before must then be re-captured)."""
        from . import _lib
        grid = _lib.relay_sys_grid(self.b, self.hq, self.hkv, self.sys_cache.system_len,
                                   int(ctx_tokens), kernels.sm_count(self.block_table.device))
        self.reorder()
        if grid == self.grid:
            return False
        self._set_grid(grid)
        return True

    def _launch(self, q, phases, out=None, k_new=None, v_new=None, slot_mapping=None):
        if q.dim() != 3 or tuple(q.shape) != (self.b, self.hq, HEAD_DIM):
            raise DimensionError(f"q must be ({self.b}, {self.hq}, {HEAD_DIM}), got {tuple(q.shape)}")
        if self._system_pending and phases & 1:
            self.ws.zero_()
        self._system_pending = phases == 1
        return kernels.relay_attention(
            q, self.q_start, self.sys_cache.keys[self.layer], self.sys_cache.values[self.layer],
            self.paged.k_pool[self.layer], self.paged.v_pool[self.layer], self.ctx_lens,
            max_rows=self.hq // self.hkv, hkv=self.hkv, sys_layout="hsd",
            block_table=self.block_table, block_size=self.paged.block_size,
            strides=self.paged.strides(), grid=self.grid, out=self.out if out is None else out,
            lse_out=self.lse, ws=self.ws, phases=phases, scale=self.scale,
            max_ctx_len=self.max_ctx_len, k_new=k_new, v_new=v_new, slot_mapping=slot_mapping,
            req_order=self.req_order)

    def system(self, q):
        """Only the system kernel of the step (profiling)."""
        return self._launch(q, 1)

    def context(self, q):
        """Only the context + fusion kernel (profiling; consumes the system
        partials of the last `system` call)."""
        return self._launch(q, 2)

    def __call__(self, q, k_new=None, v_new=None, slot_mapping=None):
        """The relay step.  With k_new / v_new (b, hkv, 128) and slot_mapping
        (int32, b): the new tokens' K / V are appended to the paged cache at
        those slots inside the same launch (the context kernel writes them
        before reading them; ctx_lens must already count them)."""
        return self._launch(q, 3, k_new=k_new, v_new=v_new, slot_mapping=slot_mapping)

    def step_host(self, q_host, k_new_host, v_new_host, slot_mapping, out_host):
        """End-to-end decode step from host buffers (pinned for async copies):
        H2D of the step's queries and new-token K/V, paged append at
        `slot_mapping` (int32 device tensor), the relay step, and D2H of the
        output into `out_host`.  All work is ordered on the current stream;
        synchronise before reading `out_host`."""
        if getattr(self, "_q_dev", None) is None:
            self._q_dev = torch.empty(q_host.shape, dtype=torch.bfloat16, device=self.out.device)
            self._k_dev = torch.empty(k_new_host.shape, dtype=torch.bfloat16, device=self.out.device)
            self._v_dev = torch.empty(v_new_host.shape, dtype=torch.bfloat16, device=self.out.device)
        self._q_dev.copy_(q_host, non_blocking=True)
        self._k_dev.copy_(k_new_host, non_blocking=True)
        self._v_dev.copy_(v_new_host, non_blocking=True)
        self.paged.append_slots(self.layer, self._k_dev, self._v_dev, slot_mapping)
        out, _ = self(self._q_dev)
        out_host.copy_(out, non_blocking=True)
        return out_host

    def host_step_graph(self, qkv_host, slot_mapping, out_host, zero_copy=True):
        """CUDA-graph version of `step_host` for a serving loop.

        qkv_host: pinned bf16 (3, b, h, 128) holding this step's q, k_new,
        v_new; out_host: pinned bf16 (b, hq, 128).  Returns a callable that
        replays the step on the current stream: the host -> device transfer
        of the inputs, the paged append of the new tokens, the relay step and
        the device -> host transfer of the output.  Refill `qkv_host` between
        calls.

        zero_copy (default): no staging copies and no separate append -- the
        two attention kernels read the queries, and the context kernel the
        new K / V (which it appends to the pool before streaming them),
        straight from the pinned host buffer over the host link (UVA); its
        fused epilogue writes the output rows straight into `out_host`.  The
        bytes crossing the link are the same as with copies.  False: one H2D
        copy, the append kernel, the step, one D2H copy (`step_host`'s order).
        """
        dev = self.out.device
        qkv_dev = torch.empty(qkv_host.shape, dtype=torch.bfloat16, device=dev)
        main = torch.cuda.current_stream(dev)

        def body():
            if zero_copy:
                # one launch pair: queries and new K / V read from the pinned
                # buffer, the append fused into the context kernel, the
                # output written into out_host
                self._launch(qkv_host[0], 3, out=out_host, k_new=qkv_host[1], v_new=qkv_host[2],
                             slot_mapping=slot_mapping)
                return
            # one H2D of [q|k_new|v_new], the paged append, then the relay step
            # (system + context kernels run concurrently; the append is the
            # system kernel's PDL primary, so its prologue overlaps it)
            qkv_dev.copy_(qkv_host, non_blocking=True)
            self.paged.append_slots(self.layer, qkv_dev[1], qkv_dev[2], slot_mapping)
            out, _ = self(qkv_dev[0])
            out_host.copy_(out, non_blocking=True)

        warm = torch.cuda.Stream(device=dev)
        warm.wait_stream(main)
        with torch.cuda.stream(warm):
            body()
        main.wait_stream(warm)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            body()
        self._host_graph = graph  # keep alive with its buffers
        self._host_graph_bufs = (qkv_dev,)
        return graph.replay


def _lib_ctx_bytes(b, hq, hkv, s_prefix, max_ctx_len, dev):
    from . import _lib
    return _lib.context_workspace_bytes(b, b, hq // hkv, hq, hkv, s_prefix, max_ctx_len,
                                        kernels.sm_count(dev))


class RelayDecodeStack:
    """The decode-attention stack of a model: one relay decode step per layer
    (the reference model's per-layer `_attend`, model.py:261-336, relay mode)
    over the layers of one SystemKvCache and one PagedKvCache, sharing the
    block table and context lengths.

    q: (layers, b, hq, 128) bf16 -> out (layers, b, hq, 128), fused lse
    (layers, b, hq).  The 2 x layers kernels are launched back to back on the
    current stream; each layer's system kernel is a programmatic dependent
    of the previous layer's context kernel, so its prologue (barriers, TMEM,
    descriptor prefetch) overlaps that kernel's tail while its first loads
    wait for it to complete.  Every layer has its own workspace, so the
    whole stack is one capturable sequence (one CUDA graph per decode step).
    """

    def __init__(self, sys_cache, paged_cache, block_table, ctx_lens, hq, grid=None,
                 out_dtype=torch.bfloat16, scale=None):
        if sys_cache.layers != paged_cache.layers:
            raise DimensionError(f"system cache has {sys_cache.layers} layers, paged cache "
                                 f"{paged_cache.layers}")
        self.layers = sys_cache.layers
        b = ctx_lens.numel()
        dev = block_table.device
        self.out = torch.empty((self.layers, b, hq, HEAD_DIM), dtype=out_dtype, device=dev)
        self.lse = torch.empty((self.layers, b, hq), dtype=torch.float32, device=dev)
        first = RelayDecodeStep(sys_cache, paged_cache, block_table, ctx_lens, hq, layer=0,
                                grid=grid, out_dtype=out_dtype, scale=scale,
                                out=self.out[0], lse=self.lse[0])
        self.steps = [first] + [
            RelayDecodeStep(sys_cache, paged_cache, block_table, ctx_lens, hq, layer=i,
                            grid=first.grid, out_dtype=out_dtype, scale=scale,
                            out=self.out[i], lse=self.lse[i])
            for i in range(1, self.layers)]
        self.grid, self.plan = first.grid, first.plan

    def __call__(self, q):
        if q.dim() != 4 or q.shape[0] != self.layers:
            raise DimensionError(f"q must be (layers={self.layers}, b, hq, 128), got {tuple(q.shape)}")
        for i, step in enumerate(self.steps):
            step(q[i])
        return self.out, self.lse


class NaiveDecodeStep:
    """The per-request baseline step ("vLLM-PS"; reference
    `baseline_attention`): every request re-reads the shared prefix (stored
    once, in the SystemKvCache) and then its own paged context, in one
    paged kernel without fusion.  Same inputs/outputs as RelayDecodeStep."""

    def __init__(self, sys_cache, paged_cache, block_table, ctx_lens, hq, layer=0,
                 out_dtype=torch.bfloat16, scale=None):
        self.sys_cache, self.paged, self.layer = sys_cache, paged_cache, layer
        self.scale = sys_cache.scale if scale is None else float(scale)
        self.block_table, self.ctx_lens = block_table, ctx_lens
        self.b = ctx_lens.numel()
        self.hq, self.hkv = hq, sys_cache.kv_heads
        dev = block_table.device
        self.out = torch.empty((self.b, hq, HEAD_DIM), dtype=out_dtype, device=dev)
        self.lse = torch.empty((self.b, hq), dtype=torch.float32, device=dev)
        self.q_start = torch.arange(self.b + 1, dtype=torch.int32, device=dev)
        self.max_ctx_len = block_table.shape[1] * paged_cache.block_size
        need = _lib_ctx_bytes(self.b, hq, self.hkv, sys_cache.system_len, self.max_ctx_len, dev)
        self.ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=dev)

    def __call__(self, q):
        pk = self.sys_cache.keys[self.layer]
        pv = self.sys_cache.values[self.layer]
        return kernels.context_attention(
            q, self.q_start, self.paged.k_pool[self.layer], self.paged.v_pool[self.layer],
            self.ctx_lens, max_rows=self.hq // self.hkv, hkv=self.hkv,
            block_table=self.block_table, block_size=self.paged.block_size,
            strides=self.paged.strides(), causal=True, prefix_k=pk, prefix_v=pv,
            prefix_strides=(pk.stride(1), pk.stride(0), pk.shape[1]),
            out=self.out, lse_out=self.lse, scale=self.scale, max_ctx_len=self.max_ctx_len,
            ws=self.ws)
