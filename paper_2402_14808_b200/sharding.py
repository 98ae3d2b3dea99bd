"""KV-head sharding of the relay decode step across the GPUs of one node.

Every (request, KV head) pair is independent in attention (the reference's
per-head loop, attention.py:122-133; fusion is per (request, query, head),
attention.py:140-141), so rank r owns a contiguous range of KV heads -- and
their g = H_q / H_kv query heads -- with that slice of the system KV and of
the paged context pool.  No collective runs inside the attention.  The only
NCCL step is `gather_heads`, an all-gather of per-rank outputs used for the
end-to-end check (outside any timed region).
"""

from __future__ import annotations

import torch


def head_ranges(hkv: int, world: int):
    """Contiguous KV-head ranges, sizes differing by at most one
    (52 heads on 8 ranks -> 7,7,7,7,6,6,6,6)."""
    if world < 1 or hkv < 1:
        raise ValueError("need world >= 1 and hkv >= 1")
    base, extra = divmod(hkv, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, start + n))
        start += n
    return out


def local_heads(hkv: int, hq: int, world: int, rank: int):
    """(kv_start, kv_end, q_start, q_end) owned by `rank`."""
    g = hq // hkv
    a, b = head_ranges(hkv, world)[rank]
    return a, b, a * g, b * g


def gather_heads(local_out: torch.Tensor, hq: int, hkv: int, group=None):
    """All-gather per-rank (rows, hq_local, d) outputs into (rows, hq, d).

    Ranks with fewer heads pad to the largest shard so all_gather_into_tensor
    moves equal-sized buffers; the padding is dropped on reassembly.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    g = hq // hkv
    ranges = head_ranges(hkv, world)
    maxh = max(b - a for a, b in ranges) * g
    rows, hl, d = local_out.shape
    send = local_out.new_zeros((maxh, rows, d))
    send[:hl] = local_out.transpose(0, 1)
    recv = local_out.new_empty((world * maxh, rows, d))
    dist.all_gather_into_tensor(recv, send.contiguous(), group=group)
    parts = []
    for r, (a, b) in enumerate(ranges):
        n = (b - a) * g
        parts.append(recv[r * maxh:r * maxh + n])
    return torch.cat(parts, 0).transpose(0, 1).contiguous()
