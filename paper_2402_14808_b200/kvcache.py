"""GPU-resident KV storage for the relay decode path.

SystemKvCache  <- /root/reference/pkg/src/relayserve/kvcache.py:36-63
    The shared system-prompt K/V, immutable after prefill.  Stored per layer
    as bf16 [hkv][s][128] ("hsd"): each KV head's prefix is one contiguous
    s x 256 B slab, so the system kernel's TMA boxes (128 keys x 64 dims)
    are dense and every byte is read exactly once per decode step.

PagedKvCache   <- kvcache.py:113-271 (block pool + PagedKvCache)
    Per-request context K/V in fixed-size blocks.  Pool layout per layer is
    bf16 [num_blocks][hkv][block_size][128]: one (block, head) pair is a
    contiguous block_size x 256 B run (4 KB at block_size 16), read in place
    by the context kernel through an int32 block table -- no gather copy
    (the reference copies to contiguous scratch, kvcache.py:237-262).
    Block accounting (BlockAllocator: an int32 free stack, per-request block
    lists) is host bookkeeping, not device work; running out of blocks
    raises CapacityError as the reference's pool does.
"""

from __future__ import annotations

import numpy as np
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

    def __init__(self, keys, values, prompt_id: str = "system", head_dim: int = HEAD_DIM):
        if len(keys) != len(values) or not keys:
            raise DimensionError("keys/values must have one entry per layer")
        shape = tuple(keys[0].shape)
        dev = keys[0].device
        for k, v in zip(keys, values):
            if tuple(k.shape) != shape or tuple(v.shape) != shape or k.dim() != 3:
                raise DimensionError(f"layer shapes inconsistent: {tuple(k.shape)} vs {tuple(v.shape)}")
            if shape[2] != HEAD_DIM:
                raise DimensionError(f"the stored head_dim must be {HEAD_DIM} (zero-padded)")
            for t in (k, v):
                if t.device != dev:
                    raise ContractError(f"system K/V layers on different devices: {dev} vs {t.device}")
        if shape[1] < 1:
            raise ContractError("system cache must hold at least one token")
        if not 1 <= head_dim <= HEAD_DIM:
            raise DimensionError(f"head_dim {head_dim} outside 1..{HEAD_DIM}")
        # bf16 is the storage type the system kernel's TMA maps describe
        self.keys = [k.to(torch.bfloat16).contiguous() for k in keys]
        self.values = [v.to(torch.bfloat16).contiguous() for v in values]
        self.prompt_id = prompt_id
        # the model's head dim: dims past it are zero padding; the softmax
        # scale of attention over this cache is head_dim ** -0.5
        self.head_dim = int(head_dim)

    @property
    def scale(self):
        return self.head_dim ** -0.5

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
        layout, kvcache.py:40-41), converting to bf16 [h][s][128] (d < 128 is
        zero-padded and recorded as the cache's head_dim)."""
        d = int(torch.as_tensor(keys_shd[0]).shape[-1])
        if d > HEAD_DIM:
            raise DimensionError(f"head_dim {d} > {HEAD_DIM} is not supported")

        def conv(x):
            t = torch.as_tensor(x).to(device=device, dtype=torch.float32)
            t = torch.nn.functional.pad(t, (0, HEAD_DIM - d)) if d < HEAD_DIM else t
            return t.to(torch.bfloat16).permute(1, 0, 2).contiguous()
        return cls([conv(k) for k in keys_shd], [conv(v) for v in values_shd], prompt_id,
                   head_dim=d)

    @classmethod
    def prefill(cls, q_layers, k_layers, v_layers, base=kernels.ROPE_BASE, prompt_id="system",
                head_dim=HEAD_DIM, out_dtype=torch.bfloat16):
        """GPU prefill of the shared system prompt (`prefill_system_cache`,
        model.py:341-353, with the attention of its prompt phase,
        model.py:314-316).  Per layer, from the model's projections of the s
        prompt tokens -- q (s, hq, 128), k / v (s, hkv, 128) bf16 CUDA, not
        yet rotated:

        * q and k rotated to positions 0..s-1 (rope_rows, model.py:292-293;
          fp64 angles) and the rotated K with V written straight into this
          cache's [hkv][s][128] layout, one launch (rb_rope_append with the
          dense cache as a single s-token block);
        * the prefill attention -- causal over the prompt, row t sees keys
          0..t (attention_with_lse(causal=True)) -- by the context kernel
          reading the new cache in place (ragged mode, split-K over long
          prompts).

        Returns (cache, [(out, lse) per layer]): out (s, hq, 128) in
        `out_dtype`, lse (s, hq) fp32 natural log."""
        if not (len(q_layers) == len(k_layers) == len(v_layers)) or len(k_layers) == 0:
            raise DimensionError("q / k / v need one entry per layer")
        keys, values, outs = [], [], []
        for q, k, v in zip(q_layers, k_layers, v_layers):
            if q.dim() != 3 or k.dim() != 3 or k.shape != v.shape or q.shape[0] != k.shape[0]:
                raise DimensionError(f"prefill expects q (s, hq, 128), k / v (s, hkv, 128); got "
                                     f"{tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
            s, hkv, hq = k.shape[0], k.shape[1], q.shape[1]
            if s < 1:
                raise ContractError("system prompt must be non-empty")
            if hq % hkv != 0:
                raise DimensionError(f"hq={hq} must be a multiple of hkv={hkv}")
            dev = k.device
            kc = torch.empty((hkv, s, HEAD_DIM), dtype=torch.bfloat16, device=dev)
            vc = torch.empty_like(kc)
            pos = torch.arange(s, dtype=torch.int64, device=dev)
            qr = kernels.rope_append(q.to(torch.bfloat16).contiguous(), k.to(torch.bfloat16).contiguous(),
                                     v.to(torch.bfloat16).contiguous(), pos, pos.to(torch.int32),
                                     kc.unsqueeze(0), vc.unsqueeze(0), s, base=base)
            out, lse = kernels.context_attention(
                qr, torch.tensor([0, s], dtype=torch.int32, device=dev), kc, vc,
                torch.tensor([s], dtype=torch.int32, device=dev), max_rows=s * (hq // hkv), hkv=hkv,
                req_offset=torch.zeros(1, dtype=torch.int64, device=dev),
                strides=(0, kc.stride(1), kc.stride(0)), causal=True, scale=head_dim ** -0.5,
                out_fp32=out_dtype == torch.float32, max_ctx_len=s)
            keys.append(kc)
            values.append(vc)
            outs.append((out if out.dtype == out_dtype else out.to(out_dtype), lse))
        return cls(keys, values, prompt_id, head_dim=head_dim), outs

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
        return cls(keys, values, prompt_id, head_dim=d)

    def save(self, path, head_dim=None, bits=32):
        """Write the reference's format (readable by its load_system_cache):
        the first `head_dim` dims of each head (default: the cache's own
        head_dim, so a loaded d=16 file saves back as d=16), as IEEE floats
        of `bits` bits (32 holds bf16 exactly)."""
        head_dim = self.head_dim if head_dim is None else head_dim
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


class BlockAllocator:
    """Physical block ids of one paged pool, handed out per request.

    Free ids live in an int32 stack (``_stack[:_top]``); a request's block
    list grows by slicing whole runs off the top, and a release pushes the
    ids back so they are reused first.  Only the token -> slot arithmetic
    matters to the kernels (they read the int32 block table in place);
    which physical id a request gets does not, and ``shuffle`` scrambles the
    free order to exercise the indirection (tests, benchmark).
    """

    def __init__(self, num_blocks, block_size=DEFAULT_BLOCK_SIZE):
        if num_blocks < 1 or block_size < 1:
            raise ContractError(f"a paged pool needs >= 1 block of >= 1 token "
                                f"(num_blocks={num_blocks}, block_size={block_size})")
        self.num_blocks = int(num_blocks)
        self.block_size = int(block_size)
        self._stack = np.arange(self.num_blocks - 1, -1, -1, dtype=np.int32)
        self._top = self.num_blocks
        self._blocks: dict = {}     # request id -> list of physical block ids
        self._reserved: dict = {}   # request id -> tokens the blocks must hold

    @property
    def free_blocks(self):
        return self._top

    @property
    def used_blocks(self):
        return self.num_blocks - self._top

    def blocks_needed(self, tokens):
        return (int(tokens) + self.block_size - 1) // self.block_size

    def shuffle(self, seed):
        """Randomise which free ids are handed out next."""
        rng = np.random.default_rng(seed)
        self._stack[:self._top] = rng.permutation(self._stack[:self._top])

    def open(self, request_id):
        if request_id in self._blocks:
            raise ContractError(f"request {request_id!r} is already open in this pool")
        self._blocks[request_id] = []
        self._reserved[request_id] = 0

    def blocks(self, request_id):
        try:
            return self._blocks[request_id]
        except KeyError:
            raise ContractError(f"request {request_id!r} is not open in this pool") from None

    def reserve(self, request_id, tokens):
        """Make the request's blocks hold at least `tokens` tokens."""
        table = self.blocks(request_id)
        short = self.blocks_needed(tokens) - len(table)
        if short > self._top:
            raise CapacityError(f"paged pool full: {short} more block(s) for {request_id!r}, "
                                f"{self._top} of {self.num_blocks} free")
        if short > 0:
            run = self._stack[self._top - short:self._top][::-1]
            self._top -= short
            table.extend(int(x) for x in run)
        self._reserved[request_id] = max(self._reserved[request_id], int(tokens))
        return self._reserved[request_id]

    def close(self, request_id):
        """Return the request's blocks to the pool (number returned)."""
        table = self._blocks.pop(request_id, None)
        self._reserved.pop(request_id, None)
        if not table:
            return 0
        n = len(table)
        self._stack[self._top:self._top + n] = np.asarray(table[::-1], dtype=np.int32)
        self._top += n
        return n


class PagedKvCache:
    """Block-paged context K/V for all layers, resident in HBM.

    k_pool / v_pool: bf16 (layers, num_blocks, hkv, block_size, 128).  Each
    request owns a list of physical blocks (BlockAllocator) shared by all
    layers and a token count per layer; token t of a request lives in block
    ``blocks[t // block_size]`` at offset ``t % block_size``.
    """

    def __init__(self, layers, kv_heads, num_blocks, block_size=DEFAULT_BLOCK_SIZE,
                 device="cuda"):
        self.allocator = BlockAllocator(num_blocks, block_size)
        self.layers = layers
        self.kv_heads = kv_heads
        shape = (layers, num_blocks, kv_heads, block_size, HEAD_DIM)
        self.k_pool = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.v_pool = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self._tokens: dict = {}     # request id -> np.int64[layers] tokens stored
        self.device = torch.device(device)

    @property
    def block_size(self):
        return self.allocator.block_size

    def register(self, request_id):
        self.allocator.open(request_id)
        self._tokens[request_id] = np.zeros(self.layers, dtype=np.int64)

    def length(self, request_id, layer=0):
        return int(self._tokens[request_id][layer])

    def release(self, request_id):
        self._tokens.pop(request_id, None)
        return self.allocator.close(request_id)

    def extend(self, request_id, n_tokens, layers=None):
        """Account `n_tokens` more tokens on `layers` (default: all) whose
        K/V are written straight into the pools by the caller (synthetic
        workloads, prefill kernels); returns the slot of each new token on
        the first of those layers."""
        idx = range(self.layers) if layers is None else list(layers)
        counts = self._tokens[request_id]
        start = int(counts[idx[0]])
        self.allocator.reserve(request_id, int(max(counts[i] for i in idx)) + n_tokens)
        for i in idx:
            counts[i] += n_tokens
        table = self.allocator.blocks(request_id)
        bs = self.block_size
        return [table[t // bs] * bs + t % bs for t in range(start, start + n_tokens)]

    def _slots(self, request_id, layer, m):
        return self.extend(request_id, m, layers=[layer])

    def append(self, request_id, layer, k, v):
        """Append (m, hkv, 128) keys/values (kvcache.py:207-235); returns the
        new length.  The scatter runs on the GPU (rb_kv_append)."""
        if k.shape != v.shape or k.dim() != 3 or tuple(k.shape[1:]) != (self.kv_heads, HEAD_DIM):
            raise DimensionError(f"append expects (m, {self.kv_heads}, {HEAD_DIM}) pairs, "
                                 f"got {tuple(k.shape)} and {tuple(v.shape)}")
        slots = self._slots(request_id, layer, k.shape[0])
        self.append_slots(layer, k, v, torch.tensor(slots, dtype=torch.int32, device=self.device))
        return self.length(request_id, layer)

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
        pos = [context_position(self.length(r, layer), s) for r in request_ids]
        slots = [self._slots(r, layer, 1)[0] for r in request_ids]
        dev = self.device
        return kernels.rope_append(
            q.to(torch.bfloat16).contiguous(), k.to(torch.bfloat16).contiguous(),
            v.to(torch.bfloat16).contiguous(), torch.tensor(pos, dtype=torch.int64, device=dev),
            torch.tensor(slots, dtype=torch.int32, device=dev), self.k_pool[layer],
            self.v_pool[layer], self.block_size, base=base)

    def block_table(self, request_ids, width=None):
        """int32 (b, width) block table on the device (unused entries 0)."""
        tables = [self.allocator.blocks(r) for r in request_ids]
        width = max(1, max(len(t) for t in tables)) if width is None else width
        bt = torch.zeros((len(tables), width), dtype=torch.int32)
        for i, t in enumerate(tables):
            bt[i, :len(t)] = torch.tensor(t, dtype=torch.int32)
        return bt.to(self.device)

    def context_lens(self, request_ids, layer=0):
        return torch.tensor([self.length(r, layer) for r in request_ids],
                            dtype=torch.int32, device=self.device)

    def strides(self):
        """(stride_block, stride_tok, stride_head) of one layer's pool."""
        p = self.k_pool[0]
        return p.stride(0), p.stride(2), p.stride(1)

    def gather(self, request_id, layer):
        """Contiguous (c, hkv, 128) copy of a request's K/V (tests/debug)."""
        c = self.length(request_id, layer)
        table = self.allocator.blocks(request_id)
        bs = self.block_size
        ks, vs = [], []
        for i in range(0, c, bs):
            blk = table[i // bs]
            take = min(bs, c - i)
            ks.append(self.k_pool[layer, blk, :, :take].transpose(0, 1))
            vs.append(self.v_pool[layer, blk, :, :take].transpose(0, 1))
        return torch.cat(ks), torch.cat(vs)
