"""Shared helpers of the -m gpu parity tests.

Tolerances (bf16 operands, fp32 accumulation, bf16 or
fp32 output; the oracle sees the same bf16 values upcast to float64):
    output  max|dO| <= 1.5e-2  and  ||dO||_2 / ||O||_2 <= 5e-3
    LSE     max|dLSE| <= 1e-3   (natural log)

Every comparison is also appended to the JSON-lines file named by
RB_PARITY_LOG (when set), so a GPU run leaves a per-case error table
(profiles/<round>/parity_*.jsonl).
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch

O_MAX, O_REL, LSE_MAX = 1.5e-2, 5e-3, 1e-3


def errs(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    dmax = float(np.abs(got - ref).max()) if got.size else 0.0
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)) if got.size else 0.0
    return dmax, rel


def log_parity(case, **fields):
    path = os.environ.get("RB_PARITY_LOG")
    if not path:
        return
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps({"case": case, **fields}) + "\n")


def assert_close(got, ref, what, lse=False, log=True):
    dmax, rel = errs(got, ref)
    print(f"{what}: max|d|={dmax:.3e} rel={rel:.3e}")
    if log:
        log_parity(what, kind="lse" if lse else "out", max_abs=dmax, rel=rel)
    if lse:
        assert dmax <= LSE_MAX, f"{what}: LSE max err {dmax}"
    else:
        assert dmax <= O_MAX and rel <= O_REL, f"{what}: max {dmax} rel {rel}"
    return dmax, rel


def dev_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


def synth_paged_problem(b, hq, hkv, s, lens, seed, block_size=16, layers=1):
    """Seeded random bf16 decode problem resident on cuda:0: a SystemKvCache
    of `layers` x [hkv][s][128], a PagedKvCache holding len(lens) requests
    (shuffled physical blocks), q (b, hq, 128)."""
    from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache
    gen = torch.Generator(device="cuda").manual_seed(seed)
    sys_cache = SystemKvCache.random(layers, hkv, s, generator=gen)
    nblk = sum(-(-c // block_size) for c in lens) + 3
    paged = PagedKvCache(layers, hkv, nblk, block_size)
    paged.k_pool.normal_(generator=gen)
    paged.v_pool.normal_(generator=gen)
    paged.allocator.shuffle(seed)
    for r, c in enumerate(lens):
        paged.register(r)
        paged.extend(r, c)
    ids = list(range(len(lens)))
    bt, cl = paged.block_table(ids), paged.context_lens(ids)
    q = torch.randn((b, hq, 128), device="cuda", generator=gen).to(torch.bfloat16)
    return q, sys_cache, paged, bt, cl


def oracle_pair(oracle, q, sys_cache, paged, layer, r, h, g):
    """Float64 oracle of decode row r, KV head h (its g query heads) over
    [system || context]: unmasked attention of the new token over all
    s + c_r keys (= the relay output and the fused LSE).  The g query heads
    of the group go in as g query rows of one head (m = g, causal=False), so
    no g-fold KV expansion is materialised."""
    sk = sys_cache.keys[layer][h].float().cpu().numpy()
    sv = sys_cache.values[layer][h].float().cpu().numpy()
    ck, cv = paged.gather(r, layer)
    k = np.concatenate([sk, ck[:, h].float().cpu().numpy()]).astype(np.float64)
    v = np.concatenate([sv, cv[:, h].float().cpu().numpy()]).astype(np.float64)
    qn = q[r, h * g:(h + 1) * g].float().cpu().numpy().astype(np.float64)   # q: (b, hq, 128)
    res = oracle.attention_with_lse(qn[None, :, None], k[None, :, None], v[None, :, None],
                                    causal=False)
    return res.output[0, :, 0], res.lse[0, :, 0]


def check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, layer, pairs, g, tag):
    """Relay step output/LSE vs the oracle on sampled (request, KV head)
    pairs; returns the worst (o_max, o_rel, lse_max)."""
    o_got, o_ref, l_got, l_ref = [], [], [], []
    outn = out.float().cpu().numpy()
    lsen = lse.float().cpu().numpy()
    for r, h in pairs:
        ro, rl = oracle_pair(oracle, q, sys_cache, paged, layer, r, h, g)
        o_got.append(outn[r, h * g:(h + 1) * g])
        o_ref.append(ro)
        l_got.append(lsen[r, h * g:(h + 1) * g])
        l_ref.append(rl)
    o_max, o_rel = assert_close(np.stack(o_got), np.stack(o_ref), f"{tag} out ({len(pairs)} pairs)")
    l_max, _ = assert_close(np.stack(l_got), np.stack(l_ref), f"{tag} lse", lse=True)
    return o_max, o_rel, l_max
