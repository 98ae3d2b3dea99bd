"""GPU prefill of the shared system prompt into the system
kernel's layout (`prefill_system_cache`, model.py:341-353).

SystemKvCache.prefill takes the model's per-layer projections of the s
prompt tokens, rotates q / k to positions 0..s-1 and writes the rotated K
and V as bf16 [hkv][s][128] in one launch, then runs the prompt's causal
attention (model.py:314-316) on the new cache.  Checked against the float64
oracle (its rope_rows is pinned bitwise to the reference's,
tests/test_oracle.py): the stored keys are the oracle's rotation rounded
once to bf16 (within one bf16 ulp), the attention output / LSE within the
bf16 envelope, and a relay decode step over the prefilled cache agrees with
the oracle too.
"""

import numpy as np
import pytest
import torch

from gpu_util import assert_close, check_sampled_pairs, dev_bf16, synth_paged_problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("s,hq,hkv", [(300, 8, 2), (700, 4, 4), (129, 16, 2)])
def test_prefill_cache_and_attention(oracle, s, hq, hkv):
    from paper_2402_14808_b200 import _lib
    from paper_2402_14808_b200.kvcache import SystemKvCache
    _lib.load()
    rng = np.random.default_rng(s + hq)
    layers = 2
    qs = [oracle.round_bf16(rng.standard_normal((s, hq, 128))) for _ in range(layers)]
    ks = [oracle.round_bf16(rng.standard_normal((s, hkv, 128))) for _ in range(layers)]
    vs = [oracle.round_bf16(rng.standard_normal((s, hkv, 128))) for _ in range(layers)]
    cache, outs = SystemKvCache.prefill([dev_bf16(x) for x in qs], [dev_bf16(x) for x in ks],
                                        [dev_bf16(x) for x in vs], out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert cache.layers == layers and cache.kv_heads == hkv and cache.system_len == s
    g = hq // hkv
    for li in range(layers):
        pos_k = np.repeat(np.arange(s), hkv)
        k_rot = oracle.rope_rows(ks[li].reshape(s * hkv, 128), pos_k, 10000.0).reshape(s, hkv, 128)
        got_k = cache.keys[li].float().cpu().numpy().transpose(1, 0, 2)
        # rotation in fp64, one rounding to bf16: within one bf16 ulp of the oracle's
        ulp = np.maximum(np.abs(k_rot), 1e-30) * 2.0 ** -7
        assert np.all(np.abs(got_k - k_rot) <= ulp), f"layer {li}: rotated keys off by > 1 ulp"
        assert np.array_equal(cache.values[li].float().cpu().numpy().transpose(1, 0, 2), vs[li])
        pos_q = np.repeat(np.arange(s), hq)
        q_rot = oracle.round_bf16(oracle.rope_rows(qs[li].reshape(s * hq, 128), pos_q, 10000.0)
                                  .reshape(s, hq, 128))
        k_use = got_k.astype(np.float64)
        ref = oracle.attention_with_lse(q_rot[None], oracle.expand_kv(k_use, g)[None],
                                        oracle.expand_kv(vs[li], g)[None], causal=True)
        out, lse = outs[li]
        assert_close(out.cpu().numpy(), ref.output[0], f"prefill s={s} g={g} layer {li}")
        assert_close(lse.cpu().numpy(), ref.lse[0], f"prefill lse s={s} g={g} layer {li}", lse=True)


def test_prefilled_cache_feeds_the_relay_step(oracle):
    """A relay decode step over a prefilled system cache (the serving flow:
    prefill once, decode many) agrees with the oracle."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(11)
    s, hq, hkv, lens = 500, 8, 2, [40, 7, 130]
    q_sys = dev_bf16(rng.standard_normal((s, hq, 128)))
    k_sys = dev_bf16(rng.standard_normal((s, hkv, 128)))
    v_sys = dev_bf16(rng.standard_normal((s, hkv, 128)))
    cache, _ = SystemKvCache.prefill([q_sys], [k_sys], [v_sys])
    q, _, paged, bt, cl = synth_paged_problem(len(lens), hq, hkv, s, lens, seed=2)
    step = RelayDecodeStep(cache, paged, bt, cl, hq, out_dtype=torch.float32)
    out, lse = step(q)
    torch.cuda.synchronize()
    pairs = [(r, h) for r in range(len(lens)) for h in range(hkv)]
    check_sampled_pairs(oracle, out, lse, q, cache, paged, 0, pairs, hq // hkv,
                        "relay step over a prefilled system cache")
