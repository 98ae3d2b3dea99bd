"""Context split-K (rb_ctx_split): long contexts with few (request, KV head)
items are cut into chunk ranges spread over the SMs and combined by the last
split in split order.  Against the float64 oracle, bitwise repeatable, and
equal (within fp32 reassociation) to the unsplit kernel."""

import numpy as np
import pytest
import torch

from gpu_util import assert_close, check_sampled_pairs, dev_bf16, synth_paged_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    from paper_2402_14808_b200 import _lib
    _lib.load()
    import paper_2402_14808_b200 as pkg
    return pkg


def test_split_plan_engages_for_long_contexts(rb):
    from paper_2402_14808_b200 import _lib, kernels
    sms = kernels.sm_count()
    # b=2, 8 KV heads, 32k context: 16 items -> split; C2 (1664 items) -> no split
    assert _lib.context_workspace_bytes(2, 2, 4, 32, 8, 0, 32768, sms) > 0
    assert _lib.context_workspace_bytes(32, 32, 1, 52, 52, 0, 128, sms) == 0


@pytest.mark.parametrize("lens,hq,hkv", [([32768, 20000], 32, 8), ([9000], 4, 4), ([5000, 17, 300], 8, 1)])
def test_relay_step_long_context_split(rb, oracle, lens, hq, hkv):
    from paper_2402_14808_b200.attention import RelayDecodeStep
    b, s = len(lens), 1000
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=sum(lens))
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq, out_dtype=torch.float32)
    out, lse = [t.clone() for t in step(q)]
    out2, lse2 = step(q)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2), "split step not deterministic"
    g = hq // hkv
    pairs = [(r, h) for r in range(b) for h in sorted({0, hkv - 1})]
    check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, 0, pairs, g,
                        f"split relay lens={lens} hq={hq} hkv={hkv}")


def test_context_attention_split_vs_unsplit(rb, oracle):
    """Standalone context attention (causal, prompt rows) with and without
    the split: both vs the oracle, and within the bf16-P envelope of each
    other (the split moves the lazy-max references, so P rounds differently)."""
    from paper_2402_14808_b200 import kernels
    rng = np.random.default_rng(5)
    hq, hkv, m = 8, 2, 3
    lens = [6000, 2500]
    q = oracle.round_bf16(rng.standard_normal((len(lens) * m, hq, 128)))
    k = [oracle.round_bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    v = [oracle.round_bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    kd, vd = dev_bf16(np.concatenate(k)), dev_bf16(np.concatenate(v))
    qd = dev_bf16(q)
    q_start = torch.tensor([0, m, 2 * m], dtype=torch.int32, device="cuda")
    req_off = torch.tensor([0, lens[0]], dtype=torch.int64, device="cuda")
    cl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    args = dict(max_rows=m * hq // hkv, hkv=hkv, req_offset=req_off,
                strides=(0, kd.stride(0), kd.stride(1)), causal=True, out_fp32=True)
    o1, l1 = kernels.context_attention(qd, q_start, kd, vd, cl, max_ctx_len=max(lens), **args)
    o1, l1 = o1.clone(), l1.clone()
    o0, l0 = kernels.context_attention(qd, q_start, kd, vd, cl, max_ctx_len=0, **args)
    torch.cuda.synchronize()
    assert (o1 - o0).abs().max().item() < 2e-3 and (l1 - l0).abs().max().item() < 1e-4
    g = hq // hkv
    for r, c in enumerate(lens):
        ref = oracle.attention_with_lse(q[r * m:(r + 1) * m][None], oracle.expand_kv(k[r], g)[None],
                                        oracle.expand_kv(v[r], g)[None], causal=True)
        assert_close(o1[r * m:(r + 1) * m].cpu().numpy(), ref.output[0], f"ctx split request {r}")
        assert_close(l1[r * m:(r + 1) * m].cpu().numpy(), ref.lse[0], f"ctx split lse {r}", lse=True)
