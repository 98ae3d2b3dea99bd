"""The unified relay step (grid 0): no system kernel; the context kernel
takes the shared prefix as items of 8 query rows (several requests) x a
range of 16-key chunks next to the context items, and each (request, head)
publishes each system part on the unit counters the context rows' relay
fusion polls, exactly as the two-kernel step's system kernel does (opt-in:
grid 0; measured slower than the two kernels on C2).  Against the float64 oracle, against the two-kernel step, and
bitwise repeatable."""

import numpy as np
import pytest
import torch

from gpu_util import assert_close, check_sampled_pairs, log_parity, synth_paged_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    from paper_2402_14808_b200 import _lib
    _lib.load()
    import paper_2402_14808_b200 as pkg
    return pkg


@pytest.mark.parametrize("b,hq,hkv,s,lens,block", [
    (32, 8, 8, 512, [128] * 32, 16),                    # g = 1, C2-like
    (5, 4, 4, 300, [7, 40, 1, 129, 300], 16),           # 5 rows: one partial 8-row tile, partial chunk
    (12, 16, 8, 5, [33, 64, 2, 90, 17, 5, 300, 1, 8, 16, 48, 77], 16),  # g = 2, prefix < 16 keys
    (9, 16, 4, 1000, [100, 3, 250, 64, 1, 17, 400, 31, 128], 32),       # g = 4, block 32
    (6, 32, 4, 700, [1, 500, 90, 16, 333, 64], 8),     # g = 8 (one tile per request), block 8
    (2, 32, 8, 900, [20000, 3000], 16),                 # long contexts: context split-K slots too
])
def test_unified_step_vs_oracle(rb, oracle, b, hq, hkv, s, lens, block):
    from paper_2402_14808_b200.attention import RelayDecodeStep
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b * 7 + s,
                                                      block_size=block)
    uni = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=0, out_dtype=torch.float32)
    assert uni.unified
    out, lse = [t.clone() for t in uni(q)]
    o2, l2 = uni(q)
    two = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=7, out_dtype=torch.float32)
    o3, l3 = two(q)
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2), "unified step not deterministic"
    g = hq // hkv
    tag = f"unified b={b} g={g} s={s}"
    assert_close(out.cpu().numpy(), o3.cpu().numpy(), tag + " vs two-kernel step", log=False)
    assert_close(lse.cpu().numpy(), l3.cpu().numpy(), tag + " lse vs two-kernel", lse=True, log=False)
    pairs = [(r, h) for r in sorted({0, b // 2, b - 1}) for h in sorted({0, hkv - 1})]
    check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, 0, pairs, g, tag)


@pytest.mark.parametrize("s", [512, 2048])
def test_unified_c2_full_size(rb, oracle, s):
    """C2 (52 heads, b=32, c=128) at s <= 2k through the unified step."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    q, sys_cache, paged, bt, cl = synth_paged_problem(32, 52, 52, s, [128] * 32, seed=5000 + s)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, 52, grid=0)
    assert step.unified, step.grid
    out, lse = [t.clone() for t in step(q)]
    o2, l2 = step(q)
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)
    pairs = [(r, h) for r in (0, 13, 31) for h in (0, 25, 51)]
    o_max, o_rel, l_max = check_sampled_pairs(oracle, out.float(), lse, q, sys_cache, paged, 0,
                                              pairs, 1, f"C2 s={s} unified")
    log_parity(f"config C2 s={s} (unified step)", kind="config", config=f"C2s{s}", grid=0,
               pairs=len(pairs), o_max_abs=o_max, o_rel=o_rel, lse_max_abs=l_max)
