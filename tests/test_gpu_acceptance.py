"""The reference's edge-case suites run against the CUDA path.

* Randomized relay exactness (/root/reference/pkg/tests/test_acceptance.py:
  37-70: 500 cases, seed 101, every request checked against the brute-force
  causal oracle over [pad || q]) -- here 240 cases with the GPU extensions
  drawn too: GQA groups g in {1, 2, 4, 8}, heterogeneous m_r through
  relay_attention_ragged, system lengths across 128-key tile edges, head
  dims 16 and 128.  Inputs are bf16-representable, so the bound is the
  bf16-P / fp32-accumulate envelope (gpu_util), not 1e-10.
* Paged decode steps with block sizes 8 / 16 / 32 / 64 (the context
  kernel's per-row cold path for block sizes that are not a multiple of 16
  and the block-table fast path for the others).
* The LSE-gap stress lse_sys - lse_ctx = +-50 (test_attention.py:132-142)
  through the FUSED relay step, where the max-subtracted merge of system
  parts and context state runs inside the context kernel.
* naive_causal_attention (attention.py:72-93) and baseline_attention_ragged
  (attention.py:266-288) called directly with ragged inputs.
"""

import math

import numpy as np
import pytest
import torch

from gpu_util import O_MAX, assert_close, dev_bf16, errs, log_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    from paper_2402_14808_b200 import _lib
    _lib.load()
    import paper_2402_14808_b200 as pkg
    return pkg


def bf16(x):
    from oracle.relay_oracle import round_bf16
    return round_bf16(x)


def _draw_case(rng):
    b = int(rng.integers(1, 9))
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([16, 128]))
    s = int(rng.choice([int(rng.integers(1, 65)), int(rng.integers(120, 140)),
                        int(rng.integers(250, 400))]))
    if rng.integers(0, 2):           # prompt phase: m_r new tokens, ragged
        m_list = [int(rng.integers(1, 9)) for _ in range(b)]
        c_list = [m + int(rng.integers(0, 40)) for m in m_list]
    else:                            # decode
        m_list = [1] * b
        c_list = [int(rng.integers(1, 300)) for _ in range(b)]
    return b, hkv, g, d, s, m_list, c_list


def test_randomized_relay_exactness(rb, oracle):
    rng = np.random.default_rng(101)
    worst_o, worst_rel, worst_l, worst_brute = 0.0, 0.0, 0.0, 0.0
    cases = 240
    for case in range(cases):
        b, hkv, g, d, s, m_list, c_list = _draw_case(rng)
        h = hkv * g
        sys_k = bf16(rng.standard_normal((s, hkv, d)))
        sys_v = bf16(rng.standard_normal((s, hkv, d)))
        ctx_k = [bf16(rng.standard_normal((c, hkv, d))) for c in c_list]
        ctx_v = [bf16(rng.standard_normal((c, hkv, d))) for c in c_list]
        q_list = [bf16(rng.standard_normal((m, h, d))) for m in m_list]
        outs, lses = rb.relay_attention_ragged(q_list, sys_k, sys_v, ctx_k, ctx_v,
                                               return_lse=True)
        ex = lambda x: oracle.expand_kv(x, g)  # noqa: E731
        ref, ref_lse = oracle.relay_attention_ragged(
            q_list, ex(sys_k), ex(sys_v), [ex(x) for x in ctx_k], [ex(x) for x in ctx_v],
            return_lse=True)
        got = np.concatenate([o.reshape(-1) for o in outs])
        want = np.concatenate([o.reshape(-1) for o in ref])
        dmax, rel = errs(got, want)
        lmax, _ = errs(np.concatenate([x.reshape(-1) for x in lses]),
                       np.concatenate([x.reshape(-1) for x in ref_lse]))
        tag = f"case {case}: b={b} hkv={hkv} g={g} d={d} s={s} m={m_list} c={c_list}"
        assert dmax <= O_MAX and rel <= 5e-3, f"{tag}: max {dmax} rel {rel}"
        assert lmax <= 1e-3, f"{tag}: lse {lmax}"
        worst_o, worst_rel, worst_l = max(worst_o, dmax), max(worst_rel, rel), max(worst_l, lmax)
        if case % 4 == 0:
            # the reference criterion itself: brute-force causal attention
            # over [pad || q] per request (test_acceptance.py:55-63)
            for r in range(b):
                w = oracle.full_sequence_check(q_list[r][None], ex(sys_k), ex(sys_v),
                                               [ex(ctx_k[r])], [ex(ctx_v[r])], outs[r][None],
                                               np.random.default_rng(case))
                worst_brute = max(worst_brute, w)
                assert w <= O_MAX, f"{tag}: brute-force oracle {w}"
    log_parity("randomized relay exactness", kind="suite", cases=cases, o_max_abs=worst_o,
               o_rel=worst_rel, lse_max_abs=worst_l, brute_force_max_abs=worst_brute)
    print(f"{cases} cases: max|dO| {worst_o:.3e} rel {worst_rel:.3e} max|dLSE| {worst_l:.3e} "
          f"brute {worst_brute:.3e}")


@pytest.mark.parametrize("block_size", [8, 16, 32, 64])
def test_paged_block_sizes(rb, oracle, block_size):
    from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep
    from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache
    rng = np.random.default_rng(500 + block_size)
    worst = 0.0
    for case in range(6):
        b = int(rng.integers(1, 12))
        hkv = int(rng.choice([1, 2, 4]))
        g = int(rng.choice([1, 4, 8]))
        hq = hkv * g
        s = int(rng.integers(1, 700))
        lens = [int(x) for x in rng.integers(1, 400, size=b)]
        q = bf16(rng.standard_normal((b, hq, 128)))
        sk = bf16(rng.standard_normal((s, hkv, 128)))
        sv = bf16(rng.standard_normal((s, hkv, 128)))
        ck = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
        cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
        nblk = sum(-(-c // block_size) for c in lens) + 2
        paged = PagedKvCache(1, hkv, nblk, block_size)
        paged.allocator.shuffle(case)
        for r in range(b):
            paged.register(r)
            paged.append(r, 0, dev_bf16(ck[r]), dev_bf16(cv[r]))
        ids = list(range(b))
        bt, cl = paged.block_table(ids), paged.context_lens(ids)
        sys_cache = SystemKvCache.from_shd([sk], [sv])
        qd = dev_bf16(q)
        out, lse = RelayDecodeStep(sys_cache, paged, bt, cl, hq, out_dtype=torch.float32)(qd)
        nout, nlse = NaiveDecodeStep(sys_cache, paged, bt, cl, hq, out_dtype=torch.float32)(qd)
        torch.cuda.synchronize()
        ex = lambda x: oracle.expand_kv(x, g)  # noqa: E731
        ref, ref_lse = oracle.relay_attention(q[:, None], ex(sk), ex(sv), [ex(x) for x in ck],
                                              [ex(x) for x in cv], return_lse=True)
        tag = f"block {block_size} case {case} b={b} hkv={hkv} g={g} s={s}"
        d1, _ = assert_close(out.cpu().numpy(), ref[:, 0], f"{tag} relay", log=False)
        assert_close(lse.cpu().numpy(), ref_lse[:, 0], f"{tag} relay lse", lse=True, log=False)
        d2, _ = assert_close(nout.cpu().numpy(), ref[:, 0], f"{tag} naive", log=False)
        assert_close(nlse.cpu().numpy(), ref_lse[:, 0], f"{tag} naive lse", lse=True, log=False)
        worst = max(worst, d1, d2)
    log_parity(f"paged block size {block_size}", kind="suite", cases=6, o_max_abs=worst)


@pytest.mark.parametrize("gap_sign", [1, -1])
def test_lse_gap_50_through_fused_step(rb, oracle, gap_sign):
    """lse_sys - lse_ctx = +-50 (test_attention.py:132-142) inside the fused
    step: the system parts and the context state meet in the context
    kernel's max-subtracted merge; the result must equal the dominant
    segment's output (alpha = 1 / (1 + e^-50) = 1 - 2e-22) and the oracle."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(60 + gap_sign)
    b, hq, hkv, s = 8, 4, 2, 600
    g = hq // hkv
    lens = [int(x) for x in rng.integers(1, 200, size=b)]
    # scores: q . k / sqrt(128) with q = a e0 (+ small noise), system keys
    # carrying +x e0 and context keys -x e0: the segment scores differ by
    # 2 a x / sqrt(128) = 50 and the LSEs by 50 +- ln(s / c_r), in the sign given
    a, x = 8.0, 50.0 * math.sqrt(128) / (2 * 8.0)
    q = 0.05 * rng.standard_normal((b, hq, 128))
    q[..., 0] = a
    q = bf16(q)
    sk = 0.05 * rng.standard_normal((s, hkv, 128))
    sk[..., 0] = gap_sign * x
    ck = []
    for c in lens:
        k = 0.05 * rng.standard_normal((c, hkv, 128))
        k[..., 0] = -gap_sign * x
        ck.append(bf16(k))
    sk = bf16(sk)
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    from paper_2402_14808_b200.kvcache import PagedKvCache
    dv = dev_bf16
    paged = PagedKvCache(1, hkv, sum(-(-c // 16) for c in lens) + 1, 16)
    paged.allocator.shuffle(7)
    for r in range(b):
        paged.register(r)
        paged.append(r, 0, dv(ck[r]), dv(cv[r]))
    ids = list(range(b))
    step = RelayDecodeStep(SystemKvCache.from_shd([sk], [sv]), paged, paged.block_table(ids),
                           paged.context_lens(ids), hq, out_dtype=torch.float32)
    out, lse = step(dv(q))
    torch.cuda.synchronize()
    ex = lambda y: oracle.expand_kv(y, g)  # noqa: E731
    ref, ref_lse = oracle.relay_attention(q[:, None], ex(sk), ex(sv), [ex(y) for y in ck],
                                          [ex(y) for y in cv], return_lse=True)
    # the oracle's segment LSEs confirm the stress: |gap| ~ 50
    outs_ctx = [oracle.attention_with_lse(q[r][None, None], ex(ck[r])[None], ex(cv[r])[None],
                                          causal=False) for r in range(b)]
    sys_res = oracle.attention_with_lse(q[None], ex(sk)[None], ex(sv)[None], causal=False)
    gap = sys_res.lse[0] - np.stack([o.lse[0, 0] for o in outs_ctx])
    assert np.all(gap * gap_sign > 40) and np.all(gap * gap_sign < 60), gap
    tag = f"lse gap {50 * gap_sign:+d} fused step"
    assert_close(out.cpu().numpy(), ref[:, 0], tag)
    assert_close(lse.cpu().numpy(), ref_lse[:, 0], tag + " lse", lse=True)
    dominant = sys_res.output[0] if gap_sign > 0 else np.stack([o.output[0, 0] for o in outs_ctx])
    assert np.abs(out.cpu().numpy() - dominant).max() <= O_MAX


def test_naive_causal_attention_api(rb, oracle):
    rng = np.random.default_rng(71)
    for l, h, d in ((1, 2, 4), (37, 4, 128), (200, 3, 16), (129, 1, 128)):
        q, k, v = (bf16(rng.standard_normal((l, h, d))) for _ in range(3))
        got = rb.naive_causal_attention(q, k, v)
        ref = oracle.naive_causal_attention(q, k, v)
        assert got.shape == ref.shape and got.dtype == np.float64
        assert_close(got, ref, f"naive_causal_attention l={l} h={h} d={d}")
    # known answers (test_attention.py:30-42)
    q = k = np.zeros((2, 1, 1))
    k = np.ones((2, 1, 1))
    v = np.asarray([1.0, 3.0]).reshape(2, 1, 1)
    assert abs(rb.naive_causal_attention(q, k, v)[1, 0, 0] - 2.0) < 1e-6
    q1, k1, v1 = (bf16(rng.standard_normal((1, 2, 4))) for _ in range(3))
    assert np.abs(rb.naive_causal_attention(q1, k1, v1) - v1).max() < 1e-6


def test_baseline_attention_ragged_direct(rb, oracle):
    rng = np.random.default_rng(72)
    h, d = 4, 128
    m_list = [1, 3, 8, 2, 1]
    n_list = [m + int(rng.integers(0, 500)) for m in m_list]
    q_list = [bf16(rng.standard_normal((m, h, d))) for m in m_list]
    fk = [bf16(rng.standard_normal((n, h, d))) for n in n_list]
    fv = [bf16(rng.standard_normal((n, h, d))) for n in n_list]
    counter = rb.TrafficCounter()
    got = rb.baseline_attention_ragged(q_list, fk, fv, counter=counter)
    ocounter = oracle.TrafficCounter()
    ref = oracle.baseline_attention_ragged(q_list, fk, fv, counter=ocounter)
    for r in range(len(m_list)):
        assert_close(got[r], ref[r], f"baseline_attention_ragged request {r}", log=False)
    assert (counter.elements_read, counter.elements_written) == \
        (ocounter.elements_read, ocounter.elements_written)
    worst = max(errs(a, b_)[0] for a, b_ in zip(got, ref))
    log_parity("baseline_attention_ragged", kind="suite", o_max_abs=worst)
