"""Standalone repro of one rb_relay_step case (for compute-sanitizer runs).
    python profiles/repro_step.py b hq hkv s c [grid] [block_size] [phases]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402
from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache  # noqa: E402

b, hq, hkv, s, c = (int(x) for x in sys.argv[1:6])
grid = int(sys.argv[6]) if len(sys.argv) > 6 and sys.argv[6] != "0" else None
bs = int(sys.argv[7]) if len(sys.argv) > 7 else 16
phases = int(sys.argv[8]) if len(sys.argv) > 8 else 3
gen = torch.Generator(device="cuda").manual_seed(1)
sysc = SystemKvCache.random(1, hkv, s, generator=gen)
paged = PagedKvCache(1, hkv, b * (-(-c // bs)), bs)
paged.k_pool.normal_(generator=gen)
paged.v_pool.normal_(generator=gen)
for r in range(b):
    paged.register(r)
    paged.pool.grow(r, c)
    paged._layer_lengths[r][0] = c
ids = list(range(b))
step = RelayDecodeStep(sysc, paged, paged.block_table(ids), paged.context_lens(ids), hq, grid=grid)
q = torch.randn((b, hq, 128), device="cuda", generator=gen).to(torch.bfloat16)
for _ in range(2):
    out, lse = step._launch(q, phases)
torch.cuda.synchronize()
print("ok", out.float().abs().max().item(), lse.min().item(), lse.max().item())
