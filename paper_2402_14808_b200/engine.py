"""Serving engine with measured B200 attention step costs.

The reference drives its serving simulator (`relayserve/serving.py:173-240`,
`_drive`) with an engine exposing one stepping surface -- `ModelEngine`
(`engine.py:88-186`, the toy model on CPU, step cost = its wall time) or
`SimulatedEngine` (`engine.py:194-271`, bookkeeping only, analytic cost).
`B200AttentionEngine` is a third engine with that surface whose steps run
the relay decode path of this package on the GPU for the live batch:

  * the shared system prompt's K/V per layer in a GPU-resident
    `SystemKvCache` (seeded synthetic values: the projections are the model
    layer, out of scope), read once per step by the system kernel (relay
    mode) or once per request by the naive kernel (baseline mode, the
    paper's vLLM-PS);
  * every request's own tokens in the paged `PagedKvCache`, appended each
    step by the fused RoPE + append kernel at the position the reference
    gives them (`kvcache.context_position`, kvcache.py:25-33);
  * prompt steps are the prompt-phase relay (m_r rows per request, causal
    context), decode steps one row per request;
  * `StepResult.wall_s` is the device time of the step's kernels (all
    layers: append + attention), measured with CUDA events, so the
    reference's `wallclock_cost` (engine.py:83-85) -- the default cost
    function of `run_batch_job` / `run_interactive_sim` -- advances the
    simulated clock by measured B200 attention time.

Admission accounting follows the reference engines: a request reserves its
worst-case blocks up front, the prefix included in baseline mode
(`ModelEngine.blocks_needed`, engine.py:124-128), which is what limits the
baseline's batch size; the kernels themselves store the prefix once.
Generated tokens are a placeholder (never END_TOKEN), as in
`SimulatedEngine`, so requests run to their generation cap.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import torch

from . import _lib, kernels
from .errors import ContractError, DimensionError
from .kvcache import (DEFAULT_BLOCK_SIZE, HEAD_DIM, PagedKvCache, SystemKvCache,
                      context_position)

PLACEHOLDER_TOKEN = 1   # never relayserve.model.END_TOKEN (0)


@dataclass
class StepResult:
    """One engine step (the fields of relayserve.engine.StepResult, engine.py:31-40)."""

    kind: str
    tokens: dict
    attn_elements: int
    cost_elements: int
    flops: float
    wall_s: float


def attention_step_elements(mode, s, new_tokens, cache_lens, d):
    """Per-layer attention traffic of a step in the reference's counter
    convention (engine.py:43-53): the prefix is charged per request in
    baseline mode, once per step in relay mode."""
    if mode == "baseline":
        return d * sum(c + 2 * m for m, c in zip(new_tokens, cache_lens))
    return d * (s + sum(cache_lens) + 7 * sum(new_tokens))


class B200AttentionEngine:
    """Engine surface of relayserve's ModelEngine / SimulatedEngine with the
    attention step executed on the B200 (see the module docstring)."""

    def __init__(self, mode, system_len, pool_blocks, *, layers=2, heads=8, kv_heads=None,
                 block_size=DEFAULT_BLOCK_SIZE, ffn_dim=None, vocab_size=256, seed=0,
                 device="cuda", out_dtype=torch.bfloat16):
        if mode not in ("baseline", "relay"):
            raise ContractError(f"unknown mode {mode!r}")
        if system_len < 1:
            raise ContractError("the engine needs a system prompt of length >= 1")
        kv_heads = heads if kv_heads is None else kv_heads
        if heads % kv_heads != 0:
            raise DimensionError(f"heads={heads} must be a multiple of kv_heads={kv_heads}")
        _lib.load()
        self.mode = mode
        self.device = torch.device(device)
        self._gen = torch.Generator(device=self.device)
        self._gen.manual_seed(seed)
        self.sys_cache = SystemKvCache.random(layers, kv_heads, system_len, device=self.device,
                                              generator=self._gen)
        self.ctx_cache = PagedKvCache(layers, kv_heads, pool_blocks, block_size, device=self.device)
        dm = heads * HEAD_DIM
        self.config = SimpleNamespace(layers=layers, heads=heads, kv_heads=kv_heads,
                                      head_dim=HEAD_DIM, model_dim=dm,
                                      ffn_dim=ffn_dim or 4 * dm, vocab_size=vocab_size)
        self.out_dtype = out_dtype
        self._reserved: dict = {}
        self.last_output = None   # (out, lse) of the last step's last layer
        self.last_q = None        # its rotated queries (rows, heads, 128)
        self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    # ------------------------------------------------------------ surface
    @property
    def system_len(self):
        return self.sys_cache.system_len

    @property
    def free_blocks(self):
        return self.ctx_cache.allocator.free_blocks

    @property
    def total_blocks(self):
        return self.ctx_cache.allocator.num_blocks

    @property
    def reserved_blocks(self):
        return sum(self._reserved.values())

    def blocks_needed(self, request):
        """Worst-case blocks if the request decodes to its cap (the prefix
        counts in baseline mode, engine.py:124-128)."""
        prefix = self.system_len if self.mode == "baseline" else 0
        tokens = prefix + request.user_len + request.max_gen - 1
        return -(-tokens // self.ctx_cache.block_size)

    def start_request(self, request):
        self.ctx_cache.register(request.id)
        self._reserved[request.id] = self.blocks_needed(request)

    def finish_request(self, request):
        self._reserved.pop(request.id, None)
        return self.ctx_cache.release(request.id)

    def prompt_step(self, requests):
        return self._run(requests, [r.user_len for r in requests], "prompt")

    def decode_step(self, requests):
        return self._run(requests, [1] * len(requests), "decode")

    # ------------------------------------------------------------- a step
    def _run(self, requests, ms, kind):
        cfg, s = self.config, self.system_len
        hq, hkv, g = cfg.heads, cfg.kv_heads, cfg.heads // cfg.kv_heads
        ids = [r.id for r in requests]
        n = sum(ms)
        dev = self.device
        # host bookkeeping and the step's synthetic projections, before the
        # timed region: new tokens' positions and slots (all layers share
        # the request's blocks), the batch's block table and lengths
        pos, slots = [], []
        for rid, m in zip(ids, ms):
            c0 = self.ctx_cache.length(rid)
            pos += [context_position(c0 + i, s) for i in range(m)]
            slots += self.ctx_cache.extend(rid, m)
        positions = torch.tensor(pos, dtype=torch.int64, device=dev)
        slot_map = torch.tensor(slots, dtype=torch.int32, device=dev)
        bt = self.ctx_cache.block_table(ids)
        ctx_lens = self.ctx_cache.context_lens(ids)
        q_start = torch.tensor([0] + list(torch.tensor(ms).cumsum(0).tolist()), dtype=torch.int32,
                               device=dev)
        max_rows = max(ms) * g
        max_ctx_len = bt.shape[1] * self.ctx_cache.block_size
        L = cfg.layers
        q = torch.randn((L, n, hq, HEAD_DIM), generator=self._gen, device=dev).to(torch.bfloat16)
        kv = torch.randn((2, L, n, hkv, HEAD_DIM), generator=self._gen, device=dev).to(torch.bfloat16)
        grid = _lib.relay_sys_grid(n, hq, hkv, s, int(sum(self.ctx_cache.length(r) for r in ids)),
                                   kernels.sm_count(dev)) if self.mode == "relay" else 0
        out = torch.empty((n, hq, HEAD_DIM), dtype=self.out_dtype, device=dev)
        lse = torch.empty((n, hq), dtype=torch.float32, device=dev)
        pool = self.ctx_cache
        # context work claimed longest request first (RelayDecodeStep's req_order)
        order = torch.argsort(ctx_lens, descending=True, stable=True).to(torch.int32) \
            if self.mode == "relay" and n > 1 else None
        e0, e1 = self._ev
        e0.record()
        for layer in range(L):
            qr = kernels.rope_append(q[layer], kv[0, layer], kv[1, layer], positions, slot_map,
                                     pool.k_pool[layer], pool.v_pool[layer], pool.block_size)
            sk, sv = self.sys_cache.keys[layer], self.sys_cache.values[layer]
            if self.mode == "relay":
                kernels.relay_attention(
                    qr, q_start, sk, sv, pool.k_pool[layer], pool.v_pool[layer], ctx_lens,
                    max_rows=max_rows, hkv=hkv, sys_layout="hsd", block_table=bt,
                    block_size=pool.block_size, strides=pool.strides(), scale=self.sys_cache.scale,
                    grid=grid, out=out, lse_out=lse, max_ctx_len=max_ctx_len, req_order=order)
            else:
                kernels.context_attention(
                    qr, q_start, pool.k_pool[layer], pool.v_pool[layer], ctx_lens,
                    max_rows=max_rows, hkv=hkv, block_table=bt, block_size=pool.block_size,
                    strides=pool.strides(), causal=True, prefix_k=sk, prefix_v=sv,
                    prefix_strides=(sk.stride(1), sk.stride(0), s), scale=self.sys_cache.scale,
                    out=out, lse_out=lse, max_ctx_len=max_ctx_len)
        e1.record()
        e1.synchronize()
        wall = e0.elapsed_time(e1) * 1e-3
        self.last_output = (out, lse)
        self.last_q = qr
        cache_lens = [self.ctx_cache.length(r) for r in ids]
        d = cfg.model_dim
        attn = L * attention_step_elements(self.mode, s, ms, cache_lens, d)
        attended = [c + s for c in cache_lens]
        flops = float(L * (8 * n * d * d + 4 * n * d * cfg.ffn_dim
                           + sum(4 * m * a * d for m, a in zip(ms, attended)))
                      + 2 * len(ids) * d * cfg.vocab_size)
        weights = L * (4 * d * d + 2 * d * cfg.ffn_dim + 2 * d) + cfg.vocab_size * d + d
        return StepResult(kind=kind, tokens={r: PLACEHOLDER_TOKEN for r in ids},
                          attn_elements=attn, cost_elements=attn + weights, flops=flops,
                          wall_s=wall)


def measured_cost(result: StepResult) -> float:
    """Step-cost function (the reference's wallclock_cost, engine.py:83-85):
    the measured device time of the step on the B200."""
    return result.wall_s


__all__ = ["B200AttentionEngine", "StepResult", "attention_step_elements", "measured_cost",
           "PLACEHOLDER_TOKEN"]
