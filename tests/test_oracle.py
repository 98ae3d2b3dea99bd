"""Pin the CPU oracle (oracle/relay_oracle.*) to the reference.

1. against tests/golden/reference_golden.npz, produced by running the
   reference itself (tests/golden/make_golden.py) -- bitwise;
2. against the reference's compiled modules (oracle/_ref, built from
   /root/reference by oracle/build.py) when present -- bitwise;
3. the reference's own known-answer tests (test_attention.py,
   test_numerics.py, test_costmodel.py) re-run on the oracle.
"""

import math
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(os.path.dirname(HERE), "oracle", "_ref")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(HERE, "golden", "reference_golden.npz"))


def _ref():
    if not os.path.isdir(os.path.join(REF_DIR, "relayserve")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import relayserve.attention as attention
    import relayserve.kernels as kernels
    return attention, kernels


def _split(g, p):
    lens = g[p + "lens"]
    off = np.concatenate([[0], np.cumsum(lens)])
    return ([g[p + "ctx_k"][off[i]:off[i + 1]] for i in range(len(lens))],
            [g[p + "ctx_v"][off[i]:off[i + 1]] for i in range(len(lens))])


def test_softmax_golden(oracle, golden):
    for i in range(3):
        p, l = oracle.softmax_lse_rows(golden[f"softmax_in_{i}"])
        assert (p == golden[f"softmax_probs_{i}"]).all()
        assert (l == golden[f"softmax_lse_{i}"]).all()


def test_attention_with_lse_golden_bitwise(oracle, golden):
    for c in (0, 1):
        r = oracle.attention_with_lse(golden[f"awl{c}_q"], golden[f"awl{c}_k"],
                                      golden[f"awl{c}_v"], bool(c))
        assert (r.output == golden[f"awl{c}_o"]).all()
        assert (r.lse == golden[f"awl{c}_lse"]).all()


@pytest.mark.parametrize("name", ["decode", "prompt", "bf16dec"])
def test_relay_golden_bitwise(oracle, golden, name):
    p = f"relay_{name}_"
    ck, cv = _split(golden, p)
    counter = oracle.TrafficCounter()
    out, lse = oracle.relay_attention(golden[p + "q"], golden[p + "sys_k"], golden[p + "sys_v"],
                                      ck, cv, counter=counter, return_lse=True)
    assert (out == golden[p + "out"]).all()
    assert (lse == golden[p + "lse"]).all()
    assert [counter.elements_read, counter.elements_written, counter.lse_elements] == \
        list(golden[p + "traffic"])
    fk = [np.concatenate([golden[p + "sys_k"], k]) for k in ck]
    fv = [np.concatenate([golden[p + "sys_v"], v]) for v in cv]
    base = oracle.baseline_attention(golden[p + "q"], fk, fv)
    assert (base == golden[p + "baseline_out"]).all()


def test_fusion_golden_bitwise(oracle, golden):
    out = oracle.relay_fusion(golden["fusion_o_sys"], golden["fusion_lse_sys"],
                              golden["fusion_o_ctx"], golden["fusion_lse_ctx"])
    assert (out == golden["fusion_out"]).all()


def test_costmodel_golden(oracle, golden):
    for b, s, c, d, nr, nb in golden["traffic_tuples"]:
        assert oracle.traffic_relay(b, s, c, d) == nr
        assert oracle.traffic_baseline(b, s, c, d) == nb
    assert oracle.theoretical_speedup(32, 2048, 128) == golden["speedup_32_2048_128"][0]
    assert abs(oracle.theoretical_speedup(32, 2048, 128) - 2178 / 199) < 1e-9


def test_kernels_bitwise_vs_compiled_reference(oracle):
    _, kernels = _ref()
    rng = np.random.default_rng(42)
    for _ in range(10):
        m, n, k = (int(x) for x in rng.integers(1, 12, size=3))
        a = rng.standard_normal((m, k)); b = rng.standard_normal((n, k))
        assert (oracle.matmul_nt(a, b) == kernels.matmul_nt(a, b)).all()
    x = rng.standard_normal((40, 7)) * 30
    assert all((u == v).all() for u, v in zip(oracle.softmax_lse_rows(x), kernels.softmax_lse_rows(x)))
    lens = rng.integers(1, 8, size=40).astype(np.int64)
    assert all((u == v).all() for u, v in
               zip(oracle.softmax_lse_prefix(x, lens), kernels.softmax_lse_prefix(x, lens)))
    q = rng.standard_normal((15, 6)); kk = rng.standard_normal((15, 6)); v = rng.standard_normal((15, 6))
    assert (oracle.naive_attention_head(q, kk, v, 6 ** -0.5)
            == kernels.naive_attention_head(q, kk, v, 6 ** -0.5)).all()


def test_relay_bitwise_vs_compiled_reference(oracle):
    attention, _ = _ref()
    rng = np.random.default_rng(101)
    for _ in range(20):
        b = int(rng.integers(1, 6)); h = int(rng.choice([1, 2, 4])); d = int(rng.choice([4, 8, 16]))
        s = int(rng.integers(1, 40))
        m = int(rng.integers(1, 4))
        lens = [int(rng.integers(m, 30)) for _ in range(b)]
        q = rng.standard_normal((b, m, h, d))
        sk = rng.standard_normal((s, h, d)); sv = rng.standard_normal((s, h, d))
        ck = [rng.standard_normal((c, h, d)) for c in lens]
        cv = [rng.standard_normal((c, h, d)) for c in lens]
        c1, c2 = oracle.TrafficCounter(), attention.TrafficCounter()
        a = oracle.relay_attention(q, sk, sv, ck, cv, counter=c1)
        r = attention.relay_attention(q, sk, sv, ck, cv, counter=c2)
        assert (a == r).all()
        assert (c1.elements_read, c1.elements_written, c1.lse_elements) == \
            (c2.elements_read, c2.elements_written, c2.lse_elements)


def test_reference_known_answers(oracle):
    # test_attention.py:30-51
    rng = np.random.default_rng(0)
    q = rng.standard_normal((1, 2, 4)); k = rng.standard_normal((1, 2, 4)); v = rng.standard_normal((1, 2, 4))
    assert np.abs(oracle.naive_causal_attention(q, k, v) - v).max() < 1e-15
    out = oracle.naive_causal_attention(np.zeros((2, 1, 1)), np.ones((2, 1, 1)),
                                        np.asarray([1.0, 3.0]).reshape(2, 1, 1))
    assert abs(out[1, 0, 0] - 2.0) < 1e-15
    # test_attention.py:70-81 identical keys: lse = ln n + q.k/sqrt(d)
    rng = np.random.default_rng(3)
    n = 6
    q = rng.standard_normal((1, 1, 1, 4)); k1 = rng.standard_normal(4); v1 = rng.standard_normal(4)
    kk = np.tile(k1, (1, n, 1, 1)).reshape(1, n, 1, 4)
    vv = np.tile(v1, (1, n, 1, 1)).reshape(1, n, 1, 4)
    res = oracle.attention_with_lse(q, kk, vv, causal=False)
    assert np.abs(res.output[0, 0, 0] - v1).max() < 1e-14
    assert abs(res.lse[0, 0, 0] - (math.log(n) + float(q[0, 0, 0] @ k1) / 2.0)) < 1e-12
    # test_attention.py:190-194 decode exactness via the pad-query oracle
    rng = np.random.default_rng(10)
    qd = rng.standard_normal((4, 1, 2, 4)); sk = rng.standard_normal((8, 2, 4)); sv = rng.standard_normal((8, 2, 4))
    ck = [rng.standard_normal((c, 2, 4)) for c in (1, 3, 5, 7)]
    cv = [rng.standard_normal((c, 2, 4)) for c in (1, 3, 5, 7)]
    out = oracle.relay_attention(qd, sk, sv, ck, cv)
    assert oracle.full_sequence_check(qd, sk, sv, ck, cv, out, rng) < 1e-10


def test_gqa_expansion_exact(oracle):
    rng = np.random.default_rng(5)
    q = rng.standard_normal((1, 3, 8, 16)); k = rng.standard_normal((1, 5, 2, 16))
    r = oracle.attention_with_lse(q, oracle.expand_kv(k, 4), oracle.expand_kv(k, 4), causal=False)
    for h in range(8):
        rh = oracle.attention_with_lse(q[:, :, h:h + 1], k[:, :, h // 4:h // 4 + 1],
                                       k[:, :, h // 4:h // 4 + 1], causal=False)
        assert (rh.output[:, :, 0] == r.output[:, :, h]).all()


def test_round_bf16(oracle):
    import torch
    x = np.random.default_rng(1).standard_normal(1000) * 10
    t = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert (oracle.round_bf16(x) == t).all()


def test_rope_golden_bitwise(oracle, golden):
    """rope_rows (_kernels_cy.pyx:80-102) at context positions index + s
    (kvcache.py:25-33) against the reference's own outputs."""
    assert (oracle.rope_rows(golden["rope_x"], golden["rope_pos"], 10000.0)
            == golden["rope_out"]).all()
    v = golden["rope_apply_v"]
    got = np.stack([oracle.rope_rows(v[None], np.asarray([p]), 10000.0)[0] for p in (0, 1, 2, 1000)])
    assert (got == golden["rope_apply_out"]).all()
    assert oracle.context_position(5, 512) == 517
    with pytest.raises(oracle.ContractError):
        oracle.context_position(-1, 3)


def test_rope_bitwise_vs_compiled_reference(oracle):
    _, kernels = _ref()
    rng = np.random.default_rng(17)
    for n, d in ((1, 2), (7, 16), (33, 128)):
        x = rng.standard_normal((n, d))
        pos = rng.integers(0, 200000, size=n).astype(np.int64)
        assert (oracle.rope_rows(x, pos, 10000.0) == kernels.rope_rows(x, pos, 10000.0)).all()


def test_rope_properties(oracle):
    # test_numerics.py:88 (position 0 is the identity), norm preservation
    rng = np.random.default_rng(4)
    x = rng.standard_normal((50, 128))
    assert (oracle.rope_rows(x, np.zeros(50, dtype=np.int64), 10000.0) == x).all()
    y = oracle.rope_rows(x, rng.integers(0, 70000, size=50), 10000.0)
    assert np.abs(np.linalg.norm(y, axis=1) - np.linalg.norm(x, axis=1)).max() < 1e-12
