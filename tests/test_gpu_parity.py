"""GPU parity of the sm_100a kernels against the float64 CPU oracle.

Every test feeds the CUDA path and the oracle the SAME bf16-representable
inputs (the oracle sees them upcast to float64) and checks, per
SURVEY.md section 8c:
    output  max|dO| <= 1.5e-2  and  ||dO||_2 / ||O||_2 <= 5e-3
    LSE     max|dLSE| <= 1e-3   (natural log)
The GPU computes with bf16 operands, fp32 accumulation / softmax and (for the
system kernel) bf16 probabilities in the P.V MMA.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

O_MAX, O_REL, LSE_MAX = 1.5e-2, 5e-3, 1e-3


def _errs(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    dmax = float(np.abs(got - ref).max())
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    return dmax, rel


def assert_close(got, ref, what, lse=False):
    dmax, rel = _errs(got, ref)
    print(f"{what}: max|d|={dmax:.3e} rel={rel:.3e}")
    if lse:
        assert dmax <= LSE_MAX, f"{what}: LSE max err {dmax}"
    else:
        assert dmax <= O_MAX and rel <= O_REL, f"{what}: max {dmax} rel {rel}"


@pytest.fixture(scope="module")
def rb():
    import paper_2402_14808_b200 as rb_pkg
    from paper_2402_14808_b200 import _lib
    _lib.load()
    return rb_pkg


def bf16(x):
    from oracle.relay_oracle import round_bf16
    return round_bf16(x)


def dev_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


# ----------------------------------------------------------- layout probe

@pytest.mark.parametrize("nq", [16, 32, 64])
def test_umma_probe_layouts(rb, nq):
    """tcgen05 operand layouts / descriptors of the system kernel on one tile."""
    from paper_2402_14808_b200 import kernels
    g = torch.Generator().manual_seed(nq)
    k = torch.randn(128, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(128, 128, generator=g).to(torch.bfloat16)
    q = torch.randn(nq, 128, generator=g).to(torch.bfloat16)
    p = torch.rand(nq, 128, generator=g).to(torch.bfloat16)
    s_out, o_out = kernels.umma_probe(k.cuda(), q.cuda(), v.cuda(), p.cuda())
    torch.cuda.synchronize()
    s_ref = k.float() @ q.float().T            # [128 keys, nq]
    o_ref = v.float().T @ p.float().T          # [128 d, nq]
    assert torch.allclose(s_out.cpu(), s_ref, atol=1e-2, rtol=1e-3), (s_out.cpu() - s_ref).abs().max()
    assert torch.allclose(o_out.cpu(), o_ref, atol=1e-2, rtol=1e-3), (o_out.cpu() - o_ref).abs().max()


# --------------------------------------------------------- system kernel

@pytest.mark.parametrize("n_rows,hq,hkv,s,grid", [
    (4, 2, 2, 200, None),        # nq 16, partial last tile
    (32, 4, 4, 1000, None),      # nq 32 (C2-like rows)
    (32, 4, 4, 1000, 5),         # forced stream-K splits (many partial slots)
    (64, 2, 2, 384, 3),          # 64 rows/head -> 2 q-tiles of 32
    (24, 8, 2, 300, 7),          # GQA g=4: 96 rows/head -> 2 q-tiles
    (1, 1, 1, 1, None),          # single key
    (64, 8, 2, 700, None),       # 256 rows/head: non-swapped 128-row kernel, 2 q-tiles
    (40, 8, 2, 300, 5),          # 160 rows/head (partial q-tile), stream-K parts
    (128, 4, 1, 129, None),      # 512 rows/head: 256-row units (two query tiles), partial key tile
    (32, 32, 8, 1000, 3),        # g=4, 128 rows/head exactly, 3 CTAs
    (75, 4, 1, 1000, 5),         # 300 rows/head: a full and a 44-row 256-row unit, stream-K parts
    (64, 16, 4, 2000, 9),        # 256 rows/head exactly, 4 units over 9 CTAs
    (160, 8, 1, 900, None),      # 1280 rows/head: 5 units round-robin / aligned
])
def test_system_attention_vs_oracle(rb, oracle, n_rows, hq, hkv, s, grid):
    from paper_2402_14808_b200 import kernels
    rng = np.random.default_rng(1000 + n_rows + s)
    q = bf16(rng.standard_normal((n_rows, hq, 128)))
    sk = bf16(rng.standard_normal((s, hkv, 128)))
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    o, lse = kernels.system_attention(dev_bf16(q), dev_bf16(sk), dev_bf16(sv), kv_layout="shd",
                                      grid=grid)
    torch.cuda.synchronize()
    g = hq // hkv
    ref = oracle.attention_with_lse(q[None], oracle.expand_kv(sk, g)[None],
                                    oracle.expand_kv(sv, g)[None], causal=False)
    assert_close(o.cpu().numpy(), ref.output[0], f"sys o {n_rows},{hq},{hkv},{s},{grid}")
    assert_close(lse.cpu().numpy(), ref.lse[0], "sys lse", lse=True)


def test_system_attention_hsd_layout_and_determinism(rb, oracle):
    from paper_2402_14808_b200 import kernels
    rng = np.random.default_rng(7)
    q = bf16(rng.standard_normal((32, 6, 128)) * 3)   # peaky logits (x3, test_attention.py:105)
    sk = bf16(rng.standard_normal((6, 777, 128)))
    sv = bf16(rng.standard_normal((6, 777, 128)))
    args = (dev_bf16(q), dev_bf16(sk), dev_bf16(sv))
    o1, l1 = kernels.system_attention(*args, kv_layout="hsd", grid=9)
    o1, l1 = o1.clone(), l1.clone()
    o2, l2 = kernels.system_attention(*args, kv_layout="hsd", grid=9)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2), "system kernel not deterministic"
    ref = oracle.attention_with_lse(q[None], sk.transpose(1, 0, 2)[None],
                                    sv.transpose(1, 0, 2)[None], causal=False)
    assert_close(o1.cpu().numpy(), ref.output[0], "sys hsd o")
    assert_close(l1.cpu().numpy(), ref.lse[0], "sys hsd lse", lse=True)


# -------------------------------------------------------- paged helpers

def make_paged(rb, ctx_k, ctx_v, hkv, block_size=16, seed=0):
    """Paged pool with shuffled block ids (exercises the indirection)."""
    from paper_2402_14808_b200.kvcache import PagedKvCache
    total_blocks = sum(-(-len(k) // block_size) for k in ctx_k) + 3
    cache = PagedKvCache(1, hkv, total_blocks, block_size, device="cuda")
    cache.allocator.shuffle(seed)
    ids = []
    for r, (k, v) in enumerate(zip(ctx_k, ctx_v)):
        cache.register(r)
        cache.append(r, 0, dev_bf16(k), dev_bf16(v))
        ids.append(r)
    return cache, cache.block_table(ids), cache.context_lens(ids)


@pytest.mark.parametrize("b,hq,hkv,s,lens", [
    (4, 4, 4, 64, [16, 9, 1, 33]),
    (32, 8, 8, 1000, [128] * 32),
    (6, 8, 2, 300, [5, 17, 64, 100, 1, 250]),   # GQA g=4
    (3, 16, 2, 129, [40, 7, 90]),               # GQA g=8
])
def test_relay_decode_step_vs_oracle(rb, oracle, b, hq, hkv, s, lens):
    from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(b * 100 + s)
    q = bf16(rng.standard_normal((b, hq, 128)))
    sk = bf16(rng.standard_normal((s, hkv, 128)))
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    ck = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    sys_cache = SystemKvCache.from_shd([sk], [sv])
    paged, bt, cl = make_paged(rb, ck, cv, hkv)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    qd = dev_bf16(q)
    out, lse = step(qd)
    naive = NaiveDecodeStep(sys_cache, paged, bt, cl, hq)
    nout, nlse = naive(qd)
    torch.cuda.synchronize()
    g = hq // hkv
    ref, ref_lse = oracle.relay_attention(
        q[:, None], oracle.expand_kv(sk, g), oracle.expand_kv(sv, g),
        [oracle.expand_kv(x, g) for x in ck], [oracle.expand_kv(x, g) for x in cv],
        return_lse=True)
    assert_close(out.float().cpu().numpy(), ref[:, 0], f"relay o b{b} s{s}")
    assert_close(lse.cpu().numpy(), ref_lse[:, 0], "relay lse", lse=True)
    assert_close(nout.float().cpu().numpy(), ref[:, 0], f"naive o b{b} s{s}")
    assert_close(nlse.cpu().numpy(), ref_lse[:, 0], "naive lse", lse=True)


# ------------------------------------------------- reference-API mirror

def _golden():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
    return np.load(path)


def _split(g, p):
    lens = g[p + "lens"]
    off = np.concatenate([[0], np.cumsum(lens)])
    ck = [g[p + "ctx_k"][off[i]:off[i + 1]] for i in range(len(lens))]
    cv = [g[p + "ctx_v"][off[i]:off[i + 1]] for i in range(len(lens))]
    return ck, cv


def test_relay_attention_api_on_reference_golden(rb):
    """relay_attention / baseline_attention through the reference-named API on
    the reference's own golden outputs (tests/golden, bf16-representable)."""
    g = _golden()
    p = "relay_bf16dec_"
    ck, cv = _split(g, p)
    counter = rb.TrafficCounter()
    out, lse = rb.relay_attention(g[p + "q"], g[p + "sys_k"], g[p + "sys_v"], ck, cv,
                                  counter=counter, return_lse=True)
    assert isinstance(out, np.ndarray) and out.dtype == np.float64
    assert_close(out, g[p + "out"], "api relay vs reference golden")
    assert_close(lse, g[p + "lse"], "api relay lse vs reference golden", lse=True)
    assert [counter.elements_read, counter.elements_written, counter.lse_elements] == \
        list(g[p + "traffic"])
    fk = [np.concatenate([g[p + "sys_k"], k]) for k in ck]
    fv = [np.concatenate([g[p + "sys_v"], v]) for v in cv]
    counter.reset()
    base = rb.baseline_attention(g[p + "q"], fk, fv, counter=counter)
    assert_close(base, g[p + "baseline_out"], "api baseline vs reference golden")
    assert [counter.elements_read, counter.elements_written] == list(g[p + "baseline_traffic"])


@pytest.mark.parametrize("name", ["decode", "prompt"])
def test_small_head_dim_cases_vs_reference_golden(rb, name):
    """d=16 reference cases (test_attention.py:190-200 shapes): head dim padded
    to 128 on the device; float64 inputs rounded to bf16, so the bound is the
    bf16 input-rounding envelope."""
    g = _golden()
    p = f"relay_{name}_"
    ck, cv = _split(g, p)
    out = rb.relay_attention(g[p + "q"], g[p + "sys_k"], g[p + "sys_v"], ck, cv)
    dmax, rel = _errs(out, g[p + "out"])
    print(f"{name}: max {dmax:.3e} rel {rel:.3e}")
    assert dmax < 5e-2 and rel < 2e-2


def test_attention_with_lse_api(rb, oracle):
    g = _golden()
    for causal in (0, 1):
        q, k, v = (bf16(g[f"awl{causal}_{x}"]) for x in "qkv")
        res = rb.attention_with_lse(q, k, v, causal=bool(causal))
        ref = oracle.attention_with_lse(q, k, v, causal=bool(causal))
        assert res.output.shape == ref.output.shape and res.lse.shape == ref.lse.shape
        assert_close(res.output, ref.output, f"awl causal={causal}")
        assert_close(res.lse, ref.lse, f"awl lse causal={causal}", lse=True)
    # single-key known answer (test_attention.py:60-68)
    q, k, v = (bf16(g[f"single_{x}"]) for x in "qkv")
    res = rb.attention_with_lse(q, k, v, causal=False)
    assert np.abs(res.output - v).max() < 1e-6
    assert abs(res.lse[0, 0, 0] - float(q[0, 0, 0] @ k[0, 0, 0]) / math.sqrt(8)) < 1e-4


def test_relay_fusion_known_answers(rb):
    g = _golden()
    out = rb.relay_fusion(g["fusion_o_sys"], g["fusion_lse_sys"], g["fusion_o_ctx"],
                          g["fusion_lse_ctx"])
    assert np.abs(out - g["fusion_out"]).max() < 1e-5
    # equal LSE -> midpoint; gap ln 3 -> 1/4; gap 50 -> o_sys (test_attention.py:115-142)
    o1 = np.ones((1, 1, 1, 1)); o0 = np.zeros((1, 1, 1, 1))
    assert abs(rb.relay_fusion(o1, np.zeros((1, 1, 1)), o0,
                               np.full((1, 1, 1), math.log(3.0)))[0, 0, 0, 0] - 0.25) < 1e-6
    assert abs(rb.relay_fusion(o1, np.full((1, 1, 1), 50.0), o0,
                               np.zeros((1, 1, 1)))[0, 0, 0, 0] - 1.0) < 1e-6
    # saturation beyond fp32 exp range must not produce NaN / inf
    big = rb.relay_fusion(o1, np.full((1, 1, 1), 200.0), o0, np.zeros((1, 1, 1)))
    assert np.isfinite(big).all() and abs(big[0, 0, 0, 0] - 1.0) < 1e-6


def test_order_independence_bitwise(rb):
    """system_first cannot change the fused output (attention.py:208-212)."""
    rng = np.random.default_rng(12)
    q = rng.standard_normal((3, 1, 2, 128)); sk = rng.standard_normal((6, 2, 128))
    ck = [rng.standard_normal((c, 2, 128)) for c in (2, 4, 6)]
    a = rb.relay_attention(q, sk, sk, ck, ck, system_first=False)
    b = rb.relay_attention(q, sk, sk, ck, ck, system_first=True)
    assert (a == b).all()


def test_prompt_phase_relay(rb, oracle):
    """m > 1 new tokens per request (f1): causal inside the context segment."""
    rng = np.random.default_rng(11)
    b, m, h, s = 2, 6, 2, 40
    q = bf16(rng.standard_normal((b, m, h, 128)))
    sk = bf16(rng.standard_normal((s, h, 128))); sv = bf16(rng.standard_normal((s, h, 128)))
    ck = [bf16(rng.standard_normal((9, h, 128))) for _ in range(b)]
    cv = [bf16(rng.standard_normal((9, h, 128))) for _ in range(b)]
    out, lse = rb.relay_attention(q, sk, sv, ck, cv, return_lse=True)
    ref, ref_lse = oracle.relay_attention(q, sk, sv, ck, cv, return_lse=True)
    assert_close(out, ref, "prompt-phase relay")
    assert_close(lse, ref_lse, "prompt-phase lse", lse=True)
    # and the brute-force pad-query oracle of test_attention.py:168-180
    worst = oracle.full_sequence_check(q, sk, sv, ck, cv, out, np.random.default_rng(0))
    assert worst < O_MAX


def test_contract_errors(rb):
    from paper_2402_14808_b200.errors import ContractError, DimensionError
    with pytest.raises(ContractError):
        rb.relay_attention(np.zeros((1, 1, 1, 2)), np.zeros((0, 1, 2)), np.zeros((0, 1, 2)),
                           [np.zeros((1, 1, 2))], [np.zeros((1, 1, 2))])
    with pytest.raises(ContractError):
        rb.attention_with_lse(np.zeros((1, 3, 1, 2)), np.zeros((1, 2, 1, 2)),
                              np.zeros((1, 2, 1, 2)), causal=True)
    with pytest.raises(DimensionError):
        rb.attention_with_lse(np.zeros((1, 1, 3, 2)), np.zeros((1, 2, 2, 2)),
                              np.zeros((1, 2, 2, 2)), causal=False)


# ------------------------------------------- full-size (BASELINE config)

def test_c2_full_size_relay_vs_naive_and_oracle_heads(rb, oracle):
    """C2 (Llama-30B shape: 52 heads, b=32, c=128) at s=8192: relay output vs
    the naive per-request kernel (full size, size-independent agreement) and
    vs the float64 oracle on a sample of 3 heads."""
    from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    b, h, s, c = 32, 52, 8192, 128
    gen = torch.Generator(device="cuda").manual_seed(5)
    sys_cache = SystemKvCache.random(1, h, s, generator=gen)
    from paper_2402_14808_b200.kvcache import PagedKvCache
    paged = PagedKvCache(1, h, b * c // 16, 16)
    paged.k_pool.normal_(generator=gen)
    paged.v_pool.normal_(generator=gen)
    for r in range(b):
        paged.register(r)
        paged.extend(r, c)
    bt, cl = paged.block_table(list(range(b))), paged.context_lens(list(range(b)))
    q = torch.randn((b, h, 128), device="cuda", generator=gen).to(torch.bfloat16)
    out, lse = RelayDecodeStep(sys_cache, paged, bt, cl, h)(q)
    nout, nlse = NaiveDecodeStep(sys_cache, paged, bt, cl, h)(q)
    torch.cuda.synchronize()
    assert_close(out.float().cpu().numpy(), nout.float().cpu().numpy(), "C2 relay vs naive")
    assert_close(lse.cpu().numpy(), nlse.cpu().numpy(), "C2 lse relay vs naive", lse=True)
    heads = [0, 25, 51]
    qn = q.float().cpu().numpy()[:, None][:, :, heads]
    sk = sys_cache.keys[0].float().cpu().numpy()[heads].transpose(1, 0, 2)
    sv = sys_cache.values[0].float().cpu().numpy()[heads].transpose(1, 0, 2)
    ck, cv = [], []
    for r in range(b):
        k_r, v_r = paged.gather(r, 0)
        ck.append(k_r.float().cpu().numpy()[:, heads]); cv.append(v_r.float().cpu().numpy()[:, heads])
    ref, ref_lse = oracle.relay_attention(qn, sk, sv, ck, cv, return_lse=True)
    assert_close(out.float().cpu().numpy()[:, heads], ref[:, 0], "C2 relay vs oracle (3 heads)")
    assert_close(lse.cpu().numpy()[:, heads], ref_lse[:, 0], "C2 lse vs oracle", lse=True)


@pytest.mark.parametrize("grid", [None, 5, 37])
def test_fused_relay_equals_two_kernel_path(rb, oracle, grid):
    """rb_relay_attention (unmerged system partials merged in the context
    epilogue) vs rb_system_attention + rb_context_attention(o_sys): same math,
    different merge order -> agree to fp32 rounding; both vs the oracle."""
    from paper_2402_14808_b200 import kernels
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(77)
    b, hq, hkv, s = 9, 12, 3, 1500
    lens = [int(x) for x in rng.integers(1, 200, size=b)]
    q = bf16(rng.standard_normal((b, hq, 128)))
    sk = bf16(rng.standard_normal((s, hkv, 128)))
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    ck = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    sys_cache = SystemKvCache.from_shd([sk], [sv])
    paged, bt, cl = make_paged(rb, ck, cv, hkv)
    qd = dev_bf16(q)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=grid, out_dtype=torch.float32)
    out, lse = step(qd)
    o_sys, lse_sys = kernels.system_attention(qd, sys_cache.keys[0], sys_cache.values[0],
                                              kv_layout="hsd", grid=grid)
    out2, lse2 = kernels.context_attention(
        qd, step.q_start, paged.k_pool[0], paged.v_pool[0], cl, max_rows=hq // hkv, hkv=hkv,
        block_table=bt, block_size=16, strides=paged.strides(), o_sys=o_sys, lse_sys=lse_sys,
        out_fp32=True)
    torch.cuda.synchronize()
    assert (out - out2).abs().max().item() < 1e-5
    assert (lse - lse2).abs().max().item() < 1e-5
    g = hq // hkv
    ref, ref_lse = oracle.relay_attention(
        q[:, None], oracle.expand_kv(sk, g), oracle.expand_kv(sv, g),
        [oracle.expand_kv(x, g) for x in ck], [oracle.expand_kv(x, g) for x in cv],
        return_lse=True)
    assert_close(out.cpu().numpy(), ref[:, 0], f"fused relay grid={grid}")
    assert_close(lse.cpu().numpy(), ref_lse[:, 0], "fused relay lse", lse=True)
    # deterministic run to run
    out3, _ = step(qd)
    torch.cuda.synchronize()
    assert torch.equal(out, out3)


def test_concurrent_step_repeats_and_phases(rb):
    """The concurrent relay step leaves its workspace rearmed: repeated steps,
    a system-only call followed by the context kernel of the same step
    (phases 1 then 2|4, and the profiling split 1 then 2) all reproduce the
    one-call step bitwise.  Other SM splits cut the stream-K units elsewhere,
    which moves the lazy-max references and so the bf16 rounding of P: they
    agree within the bf16 envelope."""
    from paper_2402_14808_b200 import kernels
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(91)
    b, hq, hkv, s = 16, 8, 4, 2000
    lens = [int(x) for x in rng.integers(1, 300, size=b)]
    q = bf16(rng.standard_normal((b, hq, 128)))
    sk = bf16(rng.standard_normal((s, hkv, 128)))
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    ck = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    sys_cache = SystemKvCache.from_shd([sk], [sv])
    paged, bt, cl = make_paged(rb, ck, cv, hkv)
    qd = dev_bf16(q)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq, out_dtype=torch.float32)
    ref, ref_lse = [t.clone() for t in step(qd)]
    for _ in range(4):
        out, lse = step(qd)
        assert torch.equal(out, ref) and torch.equal(lse, ref_lse)
    for phases in (2 | 4, 2):
        step._launch(qd, 1)
        out, lse = step._launch(qd, phases)
        torch.cuda.synchronize()
        assert torch.equal(out, ref) and torch.equal(lse, ref_lse), f"phases 1 then {phases}"
    for grid in (1, 7, kernels.sm_count(qd.device)):
        other = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=grid, out_dtype=torch.float32)
        out, lse = other(qd)
        torch.cuda.synchronize()
        assert_close(out.cpu().numpy(), ref.cpu().numpy(), f"relay split grid={grid}")
        assert_close(lse.cpu().numpy(), ref_lse.cpu().numpy(), f"relay lse grid={grid}", lse=True)


# ------------------------------------------------- RoPE + KV append (8f2)

def test_rope_rows_vs_oracle(rb, oracle):
    """rb_rope_rows against the reference's rope_rows on the golden rows
    (positions up to 131136) and random fp32 rows of several widths."""
    from paper_2402_14808_b200 import kernels
    g = np.load(__file__.replace("test_gpu_parity.py", "golden/reference_golden.npz"))
    cases = [(g["rope_x"].astype(np.float32), g["rope_pos"])]
    rng = np.random.default_rng(23)
    for n, d in ((5, 2), (64, 16), (300, 128)):
        cases.append((rng.standard_normal((n, d)).astype(np.float32),
                      rng.integers(0, 140000, size=n).astype(np.int64)))
    for x, pos in cases:
        got = kernels.rope_rows(torch.from_numpy(x).cuda(), torch.from_numpy(pos))
        torch.cuda.synchronize()
        ref = oracle.rope_rows(x.astype(np.float64), pos, 10000.0)
        err = np.abs(got.cpu().numpy().astype(np.float64) - ref).max()
        print(f"rope rows {x.shape}: max|d| = {err:.3e}")
        assert err <= 2e-6 * max(1.0, np.abs(ref).max())


def test_rope_append_vs_oracle(rb, oracle):
    """rb_rope_append: rotated q (in place) and rotated K / raw V in the
    shuffled paged pool, against the oracle on the same bf16 inputs (output
    rounded once to bf16: at most one bf16 ulp from the rounded oracle)."""
    from paper_2402_14808_b200 import kernels
    rng = np.random.default_rng(29)
    n_tok, hq, hkv, bs, nblk = 37, 8, 2, 16, 40
    q = bf16(rng.standard_normal((n_tok, hq, 128)))
    k = bf16(rng.standard_normal((n_tok, hkv, 128)))
    v = bf16(rng.standard_normal((n_tok, hkv, 128)))
    pos = np.asarray([oracle.context_position(int(t), int(s)) for t, s in
                      zip(rng.integers(0, 4096, size=n_tok), rng.integers(0, 65536, size=n_tok))],
                     dtype=np.int64)
    slots = rng.permutation(nblk * bs)[:n_tok].astype(np.int32)
    kp = torch.zeros((nblk, hkv, bs, 128), dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros_like(kp)
    qd = dev_bf16(q)
    out = kernels.rope_append(qd, dev_bf16(k), dev_bf16(v), torch.from_numpy(pos),
                              torch.from_numpy(slots).cuda(), kp, vp, bs, q_out=qd)
    torch.cuda.synchronize()
    assert out.data_ptr() == qd.data_ptr()

    def ulps(got, ref):
        r = oracle.round_bf16(ref)
        ulp = np.maximum(np.abs(r), 1e-30) * 2.0 ** -7
        return float((np.abs(got - r) / ulp).max())

    q_ref = oracle.rope_rows(q.reshape(-1, 128), np.repeat(pos, hq), 10000.0).reshape(q.shape)
    assert ulps(qd.float().cpu().numpy(), q_ref) <= 1.0
    k_ref = oracle.rope_rows(k.reshape(-1, 128), np.repeat(pos, hkv), 10000.0).reshape(k.shape)
    kpn, vpn = kp.float().cpu().numpy(), vp.float().cpu().numpy()
    for t, sl in enumerate(slots):
        blk, off = divmod(int(sl), bs)
        assert ulps(kpn[blk, :, off], k_ref[t]) <= 1.0
        assert (vpn[blk, :, off] == v[t]).all()


def test_append_rotated_decode_prologue(rb, oracle):
    """PagedKvCache.append_rotated: each request's new token lands after its
    context at position c_r + s, K rotated in the pool, q returned rotated."""
    from paper_2402_14808_b200.kvcache import PagedKvCache
    rng = np.random.default_rng(31)
    b, hq, hkv, s = 5, 4, 2, 1000
    cache = PagedKvCache(2, hkv, 64, 16, device="cuda")
    ids = [f"r{i}" for i in range(b)]
    lens = [int(x) for x in rng.integers(0, 40, size=b)]
    for r, c in zip(ids, lens):
        cache.register(r)
        if c:
            cache.append(r, 1, dev_bf16(rng.standard_normal((c, hkv, 128))),
                         dev_bf16(rng.standard_normal((c, hkv, 128))))
    q = bf16(rng.standard_normal((b, hq, 128)))
    k = bf16(rng.standard_normal((b, hkv, 128)))
    v = bf16(rng.standard_normal((b, hkv, 128)))
    qr = cache.append_rotated(ids, 1, dev_bf16(q), dev_bf16(k), dev_bf16(v), s)
    torch.cuda.synchronize()
    pos = np.asarray([c + s for c in lens], dtype=np.int64)
    q_ref = oracle.round_bf16(oracle.rope_rows(q.reshape(-1, 128), np.repeat(pos, hq), 10000.0))
    assert np.abs(qr.float().cpu().numpy().reshape(-1, 128) - q_ref).max() <= 2.0 ** -6 * np.abs(q_ref).max()
    for i, (r, c) in enumerate(zip(ids, lens)):
        assert cache.length(r, 1) == c + 1
        kk, vv = cache.gather(r, 1)
        k_ref = oracle.round_bf16(oracle.rope_rows(k[i], np.full(hkv, pos[i]), 10000.0))
        assert np.abs(kk[c].float().cpu().numpy() - k_ref).max() <= 2.0 ** -6 * np.abs(k_ref).max()
        assert (vv[c].float().cpu().numpy() == v[i]).all()


@pytest.mark.parametrize("b,s", [(48, 900), (40, 100), (80, 1300), (130, 257)])
def test_relay_step_gqa_large_vs_oracle(rb, oracle, b, s):
    """The concurrent relay step with >= 128 rows per KV head (the non-swapped
    system kernel's parts fused in the context kernel) against the oracle,
    and bitwise repeatable; s=100 gives one-tile units."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from paper_2402_14808_b200.kvcache import SystemKvCache
    rng = np.random.default_rng(77 + s)
    hq, hkv = 8, 2
    lens = [int(x) for x in rng.integers(1, 160, size=b)]
    q = bf16(rng.standard_normal((b, hq, 128)))
    sk = bf16(rng.standard_normal((s, hkv, 128)))
    sv = bf16(rng.standard_normal((s, hkv, 128)))
    ck = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    cv = [bf16(rng.standard_normal((c, hkv, 128))) for c in lens]
    paged, bt, cl = make_paged(rb, ck, cv, hkv)
    qd = dev_bf16(q)
    for grid in (None, 3):
        step = RelayDecodeStep(SystemKvCache.from_shd([sk], [sv]), paged, bt, cl, hq, grid=grid,
                               out_dtype=torch.float32)
        out, lse = [t.clone() for t in step(qd)]
        o2, l2 = step(qd)
        torch.cuda.synchronize()
        assert torch.equal(out, o2) and torch.equal(lse, l2)
        g = hq // hkv
        for r in (0, 17, b - 1):
            fk = oracle.expand_kv(np.concatenate([sk, ck[r]]), g)
            fv = oracle.expand_kv(np.concatenate([sv, cv[r]]), g)
            ref = oracle.attention_with_lse(q[r][None, None], fk[None], fv[None], causal=False)
            assert_close(out[r].cpu().numpy(), ref.output[0, 0], f"relay gqa-large row {r} grid {grid}")
            assert_close(lse[r].cpu().numpy(), ref.lse[0, 0], "relay gqa-large lse", lse=True)


@pytest.mark.parametrize("b,hq,hkv,s,grid,nq", [
    (48, 32, 8, 600, 16, 128),     # 192 rows / head: 128-row kernel, 16 units round-robin
    (128, 32, 8, 700, 16, 256),    # 512 rows / head: 256-row kernel, 16 units round-robin
    (256, 64, 8, 300, 64, 256),    # C5's head layout at s=300: 64 units, one CTA each
])
def test_relay_step_round_robin_units(rb, oracle, b, hq, hkv, s, grid, nq):
    """Whole units dealt round-robin (plan rr = 1: one part per unit, the
    CTAs of a head's units walk its key tiles in lockstep) through the relay
    step, for both GQA system kernels, against the oracle."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    from gpu_util import check_sampled_pairs, synth_paged_problem
    lens = [int(x) for x in np.random.default_rng(b + s).integers(1, 200, size=b)]
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b * s)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=grid, out_dtype=torch.float32)
    assert step.plan["rr"] == 1 and step.plan["nq"] == nq, step.plan
    out, lse = [t.clone() for t in step(q)]
    o2, l2 = step(q)
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)
    g = hq // hkv
    pairs = [(0, 0), (b // 2, hkv // 2), (b - 1, hkv - 1)]
    check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, 0, pairs, g,
                        f"rr relay nq={nq} b={b} grid={grid}")


def test_relaykv_cache_feeds_system_kernel(rb, oracle):
    """A reference-written RELAYKV file (d=16, float32) loaded straight to
    the GPU layout drives the system kernel: zero-padded head dims keep the
    attention exact against the oracle on the file's own values."""
    import os
    from paper_2402_14808_b200 import kernels
    from paper_2402_14808_b200.kvcache import SystemKvCache
    here = os.path.dirname(os.path.abspath(__file__))
    cache = SystemKvCache.load(os.path.join(here, "golden", "system_f32.relaykv"))
    g = np.load(os.path.join(here, "golden", "reference_golden.npz"))
    rng = np.random.default_rng(12)
    q16 = bf16(rng.standard_normal((5, 3, 16)))
    q = np.zeros((5, 3, 128))
    q[:, :, :16] = q16
    o, lse = kernels.system_attention(dev_bf16(q), cache.keys[1], cache.values[1], kv_layout="hsd",
                                      scale=16 ** -0.5)
    torch.cuda.synchronize()
    k = bf16(g["relaykv_f32_keys"][1])
    v = bf16(g["relaykv_f32_values"][1])
    ref = oracle.attention_with_lse(q16[None], k[None], v[None], causal=False)
    assert_close(o.cpu().numpy()[:, :, :16], ref.output[0], "relaykv sys o")
    assert np.abs(o.cpu().numpy()[:, :, 16:]).max() == 0
    assert_close(lse.cpu().numpy(), ref.lse[0], "relaykv sys lse", lse=True)
