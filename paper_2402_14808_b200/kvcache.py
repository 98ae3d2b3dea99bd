"""GPU-resident KV storage for the relay decode path.

SystemKvCache  <- /root/reference/pkg/src/relayserve/kvcache.py:36-63
    The shared system-prompt K/V, immutable after prefill.  Stored per layer
    as bf16 [hkv][s][128] ("hsd"): each KV head's prefix is one contiguous
    s x 256 B slab, so the system kernel's TMA boxes (128 keys x 64 dims)
    are dense and every byte is read exactly once per decode step.

PagedKvCache   <- kvcache.py:113-271 (BlockPool + PagedKvCache)
    Per-request context K/V in fixed-size blocks.  Pool layout per layer is
    bf16 [num_blocks][hkv][block_size][128]: one (block, head) pair is a
    contiguous block_size x 256 B run (4 KB at block_size 16), read in place
    by the context kernel through an int32 block table -- no gather copy
    (the reference copies to contiguous scratch, kvcache.py:237-262).
    Block accounting (register / grow / release, CapacityError) follows
    BlockPool exactly; it is host bookkeeping, not device work.
"""

from __future__ import annotations

import torch

from . import kernels
from .errors import CapacityError, ContractError, DimensionError

DEFAULT_BLOCK_SIZE = 16
HEAD_DIM = kernels.HEAD_DIM


def context_position(token_index_in_context: int, s: int) -> int:
    """kvcache.py:25-33: absolute position of a context token after a shared
    prefix of length s."""
    if token_index_in_context < 0:
        raise ContractError(f"token index must be >= 0, got {token_index_in_context}")
    if s < 0:
        raise ContractError(f"prefix length must be >= 0, got {s}")
    return token_index_in_context + s


class SystemKvCache:
    """Shared prefix K/V per layer, bf16 [hkv][s][128] on one device."""

    def __init__(self, keys, values, prompt_id: str = "system"):
        if len(keys) != len(values) or not keys:
            raise DimensionError("keys/values must have one entry per layer")
        shape = tuple(keys[0].shape)
        for k, v in zip(keys, values):
            if tuple(k.shape) != shape or tuple(v.shape) != shape or k.dim() != 3:
                raise DimensionError(f"layer shapes inconsistent: {tuple(k.shape)} vs {tuple(v.shape)}")
            if shape[2] != HEAD_DIM:
                raise DimensionError(f"head_dim must be {HEAD_DIM}")
        if shape[1] < 1:
            raise ContractError("system cache must hold at least one token")
        self.keys = [k.contiguous() for k in keys]
        self.values = [v.contiguous() for v in values]
        self.prompt_id = prompt_id

    @property
    def layers(self):
        return len(self.keys)

    @property
    def kv_heads(self):
        return self.keys[0].shape[0]

    @property
    def system_len(self):
        return self.keys[0].shape[1]

    @classmethod
    def from_shd(cls, keys_shd, values_shd, device="cuda", prompt_id="system"):
        """Build from per-layer (s, h, d) arrays/tensors (the reference's
        layout, kvcache.py:40-41), converting to bf16 [h][s][d]."""
        def conv(x):
            t = torch.as_tensor(x)
            return t.to(device=device, dtype=torch.bfloat16).permute(1, 0, 2).contiguous()
        return cls([conv(k) for k in keys_shd], [conv(v) for v in values_shd], prompt_id)

    # ---- the reference's on-disk format (RELAYKV, kvcache.py:19-20, 66-100):
    # magic b"RELAYKV\0", little-endian uint32 version (1), layers, s, h, d,
    # bits; then per layer the K tensor and the V tensor, (s, h, d) row-major
    # little-endian IEEE floats of `bits` bits.
    _MAGIC = b"RELAYKV\x00"
    _VERSION = 1

    @classmethod
    def load(cls, path, device="cuda", prompt_id="system"):
        """Read a file written by the reference's save_system_cache (or by
        `save`) straight into GPU-resident bf16 [h][s][128] (head dims < 128
        are zero-padded, which leaves attention exact)."""
        import struct

        import numpy as np
        with open(path, "rb") as f:
            if f.read(len(cls._MAGIC)) != cls._MAGIC:
                raise ContractError(f"{path}: not a system KV cache file")
            version, layers, s, h, d, bits = struct.unpack("<IIIIII", f.read(24))
            if version != cls._VERSION:
                raise ContractError(f"{path}: unsupported version {version}")
            if bits not in (16, 32, 64):
                raise ContractError(f"{path}: unsupported precision {bits} bits")
            if d > HEAD_DIM or d < 1:
                raise DimensionError(f"{path}: head_dim {d} unsupported (kernels take <= {HEAD_DIM})")
            dtype = np.dtype(f"<f{bits // 8}")
            count = s * h * d
            keys, values = [], []
            for _ in range(layers):
                for out in (keys, values):
                    raw = f.read(count * dtype.itemsize)
                    if len(raw) != count * dtype.itemsize:
                        raise ContractError(f"{path}: truncated")
                    a = np.frombuffer(raw, dtype=dtype).astype(np.float32).reshape(s, h, d)
                    t = torch.zeros((h, s, HEAD_DIM), dtype=torch.bfloat16, device=device)
                    t[:, :, :d] = torch.from_numpy(a).to(device).permute(1, 0, 2).to(torch.bfloat16)
                    out.append(t)
        return cls(keys, values, prompt_id)

    def save(self, path, head_dim=HEAD_DIM, bits=32):
        """Write the reference's format (readable by its load_system_cache):
        the first `head_dim` dims of each head, as IEEE floats of `bits` bits
        (32 holds bf16 exactly)."""
        import struct

        import numpy as np
        if bits not in (16, 32, 64):
            raise ContractError(f"unsupported precision {bits} bits")
        h, s, _ = self.keys[0].shape
        header = self._MAGIC + struct.pack("<IIIIII", self._VERSION, self.layers, s, h, head_dim, bits)
        with open(path, "wb") as f:
            f.write(header)
            for k, v in zip(self.keys, self.values):
                for t in (k, v):
                    a = t[:, :, :head_dim].permute(1, 0, 2).float().cpu().numpy()
                    f.write(np.ascontiguousarray(a).astype(f"<f{bits // 8}").tobytes())

    @classmethod
    def random(cls, layers, kv_heads, s, device="cuda", generator=None, prompt_id="system"):
        keys = [torch.randn((kv_heads, s, HEAD_DIM), device=device, generator=generator,
                            dtype=torch.float32).to(torch.bfloat16) for _ in range(layers)]
        values = [torch.randn((kv_heads, s, HEAD_DIM), device=device, generator=generator,
                              dtype=torch.float32).to(torch.bfloat16) for _ in range(layers)]
        return cls(keys, values, prompt_id)


class BlockPool:
    """Bookkeeping-only block allocator, same semantics as kvcache.py:113-172."""

    def __init__(self, num_blocks, block_size=DEFAULT_BLOCK_SIZE):
        if num_blocks < 1 or block_size < 1:
            raise ContractError("pool needs at least one block of one slot")
        self.num_blocks = num_blocks
        self.block_size = block_size
        self._free = list(range(num_blocks - 1, -1, -1))
        self.tables: dict = {}
        self.lengths: dict = {}

    @property
    def free_blocks(self):
        return len(self._free)

    @property
    def used_blocks(self):
        return self.num_blocks - len(self._free)

    def blocks_for(self, tokens):
        return -(-tokens // self.block_size)

    def register(self, request_id):
        if request_id in self.tables:
            raise ContractError(f"request {request_id!r} already registered")
        self.tables[request_id] = []
        self.lengths[request_id] = 0

    def grow(self, request_id, n_tokens):
        if request_id not in self.tables:
            raise ContractError(f"unknown request {request_id!r}")
        table = self.tables[request_id]
        new_len = self.lengths[request_id] + n_tokens
        need = self.blocks_for(new_len)
        if need - len(table) > len(self._free):
            raise CapacityError(
                f"pool exhausted: request {request_id!r} needs {need - len(table)} blocks, "
                f"{len(self._free)} free")
        while len(table) < need:
            table.append(self._free.pop())
        self.lengths[request_id] = new_len
        return new_len

    def release(self, request_id):
        table = self.tables.pop(request_id, [])
        self.lengths.pop(request_id, None)
        for bid in reversed(table):
            self._free.append(bid)
        return len(table)


class PagedKvCache:
    """Block-paged context K/V for all layers, resident in HBM.

    k_pool / v_pool: bf16 (layers, num_blocks, hkv, block_size, 128).
    """

    def __init__(self, layers, kv_heads, num_blocks, block_size=DEFAULT_BLOCK_SIZE,
                 device="cuda"):
        self.pool = BlockPool(num_blocks, block_size)
        self.layers = layers
        self.kv_heads = kv_heads
        shape = (layers, num_blocks, kv_heads, block_size, HEAD_DIM)
        self.k_pool = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.v_pool = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self._layer_lengths: dict = {}
        self.device = torch.device(device)

    @property
    def block_size(self):
        return self.pool.block_size

    def register(self, request_id):
        self.pool.register(request_id)
        self._layer_lengths[request_id] = [0] * self.layers

    def length(self, request_id, layer=0):
        return self._layer_lengths[request_id][layer]

    def release(self, request_id):
        self._layer_lengths.pop(request_id, None)
        return self.pool.release(request_id)

    def _slots(self, request_id, layer, m):
        lengths = self._layer_lengths[request_id]
        start = lengths[layer]
        table = self.pool.tables[request_id]
        if self.pool.blocks_for(start + m) > len(table):
            self.pool.grow(request_id, (start + m) - self.pool.lengths[request_id])
        bs = self.block_size
        slots = [table[(start + t) // bs] * bs + (start + t) % bs for t in range(m)]
        lengths[layer] = start + m
        return slots

    def append(self, request_id, layer, k, v):
        """Append (m, hkv, 128) keys/values (kvcache.py:207-235); returns the
        new length.  The scatter runs on the GPU (rb_kv_append)."""
        if k.shape != v.shape or k.dim() != 3 or tuple(k.shape[1:]) != (self.kv_heads, HEAD_DIM):
            raise DimensionError(f"append expects (m, {self.kv_heads}, {HEAD_DIM}) pairs, "
                                 f"got {tuple(k.shape)} and {tuple(v.shape)}")
        slots = self._slots(request_id, layer, k.shape[0])
        self.append_slots(layer, k, v, torch.tensor(slots, dtype=torch.int32, device=self.device))
        return self._layer_lengths[request_id][layer]

    def append_slots(self, layer, k, v, slot_mapping):
        """Device-side append with a precomputed int32 slot mapping."""
        if k.dtype != torch.bfloat16 or not k.is_contiguous():
            k = k.to(torch.bfloat16).contiguous()
        if v.dtype != torch.bfloat16 or not v.is_contiguous():
            v = v.to(torch.bfloat16).contiguous()
        kernels.kv_append(k, v, slot_mapping, self.k_pool[layer], self.v_pool[layer],
                          self.block_size)

    def append_rotated(self, request_ids, layer, q, k, v, s, base=kernels.ROPE_BASE):
        """Decode-step prologue for one new token per request: rotate q and k
        to the token's absolute position context_position(c_r, s) (the token
        lands after the request's c_r context tokens and the s-token shared
        prefix, kvcache.py:25-33; model.py:292-293) and append the rotated K
        and raw V (kvcache.py:207-235), in one launch.  q (b, hq, 128), k / v
        (b, hkv, 128) bf16; returns the rotated q."""
        if k.shape != v.shape or k.dim() != 3 or tuple(k.shape[1:]) != (self.kv_heads, HEAD_DIM):
            raise DimensionError(f"append expects (b, {self.kv_heads}, {HEAD_DIM}) pairs, "
                                 f"got {tuple(k.shape)} and {tuple(v.shape)}")
        if q.shape[0] != len(request_ids) or k.shape[0] != len(request_ids):
            raise DimensionError("append_rotated: one token per request")
        pos = [context_position(self._layer_lengths[r][layer], s) for r in request_ids]
        slots = [self._slots(r, layer, 1)[0] for r in request_ids]
        dev = self.device
        return kernels.rope_append(
            q.to(torch.bfloat16).contiguous(), k.to(torch.bfloat16).contiguous(),
            v.to(torch.bfloat16).contiguous(), torch.tensor(pos, dtype=torch.int64, device=dev),
            torch.tensor(slots, dtype=torch.int32, device=dev), self.k_pool[layer],
            self.v_pool[layer], self.block_size, base=base)

    def block_table(self, request_ids, width=None):
        """int32 (b, width) block table on the device (unused entries 0)."""
        tables = [self.pool.tables[r] for r in request_ids]
        width = max(1, max(len(t) for t in tables)) if width is None else width
        bt = torch.zeros((len(tables), width), dtype=torch.int32)
        for i, t in enumerate(tables):
            bt[i, :len(t)] = torch.tensor(t, dtype=torch.int32)
        return bt.to(self.device)

    def context_lens(self, request_ids, layer=0):
        return torch.tensor([self._layer_lengths[r][layer] for r in request_ids],
                            dtype=torch.int32, device=self.device)

    def strides(self):
        """(stride_block, stride_tok, stride_head) of one layer's pool."""
        p = self.k_pool[0]
        return p.stride(0), p.stride(2), p.stride(1)

    def gather(self, request_id, layer):
        """Contiguous (c, hkv, 128) copy of a request's K/V (tests/debug)."""
        c = self._layer_lengths[request_id][layer]
        table = self.pool.tables[request_id]
        bs = self.block_size
        ks, vs = [], []
        for i in range(0, c, bs):
            blk = table[i // bs]
            take = min(bs, c - i)
            ks.append(self.k_pool[layer, blk, :, :take].transpose(0, 1))
            vs.append(self.v_pool[layer, blk, :, :take].transpose(0, 1))
        return torch.cat(ks), torch.cat(vs)
