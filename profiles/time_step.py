"""Event-timed relay step (phases 3/1/2) for one config, L2 flushed.
    python profiles/time_step.py b hq hkv s c block_size
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep  # noqa: E402
from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache  # noqa: E402

b, hq, hkv, s, c, bs = (int(x) for x in sys.argv[1:7])
dev = torch.device("cuda", 0)
gen = torch.Generator(device="cuda").manual_seed(1)
sysc = SystemKvCache.random(1, hkv, s, generator=gen)
paged = PagedKvCache(1, hkv, b * (-(-c // bs)), bs)
paged.k_pool.normal_(generator=gen)
paged.v_pool.normal_(generator=gen)
for r in range(b):
    paged.register(r)
    paged.extend(r, c)
ids = list(range(b))
step = RelayDecodeStep(sysc, paged, paged.block_table(ids), paged.context_lens(ids), hq)
q = torch.randn((b, hq, 128), device="cuda", generator=gen).to(torch.bfloat16)
flush = bench.make_flush(torch, dev)
res = {}
for ph in (3, 1, 2):
    ms = bench.time_loop(torch, lambda: step._launch(q, ph), 20, 3, flush)
    res[ph] = statistics.mean(ms) * 1e3
print(f"b={b} hq={hq} hkv={hkv} s={s} c={c} bs={bs}: step {res[3]:.1f} us, sys-only {res[1]:.1f}, ctx-only {res[2]:.1f}")
