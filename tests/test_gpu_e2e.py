"""The end-to-end decode step from host buffers (the bench's `e2e` path):
`RelayDecodeStep.step_host` (eager) and `host_step_graph` (CUDA graph) copy
the step's q / new-token K / V from pinned memory, append the new tokens to
the paged cache, run the relay step and copy the output back.  Both must
equal the device-resident path bitwise (same kernels, same inputs) and the
float64 oracle on the appended cache."""

import numpy as np
import pytest
import torch

from gpu_util import check_sampled_pairs, synth_paged_problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b,hq,hkv,s,lens", [(6, 8, 8, 700, [33, 1, 64, 17, 100, 5]),
                                             (4, 16, 4, 300, [40, 16, 7, 90])])
def test_host_step_equals_device_step(oracle, b, hq, hkv, s, lens):
    from paper_2402_14808_b200.attention import RelayDecodeStep
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b + s)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    g = torch.Generator().manual_seed(5)
    qkv = torch.randn((3, b, hq, 128), generator=g).to(torch.bfloat16)
    qkv_h = torch.empty((3, b, hq, 128), dtype=torch.bfloat16).pin_memory()
    qkv_h[0] = qkv[0]
    qkv_h[1, :, :hkv] = qkv[1, :, :hkv]
    qkv_h[2, :, :hkv] = qkv[2, :, :hkv]
    # the new token overwrites each request's last context slot (length unchanged)
    btc = bt.cpu()
    slots = torch.tensor([int(btc[r, (c - 1) // 16]) * 16 + (c - 1) % 16 for r, c in enumerate(lens)],
                         dtype=torch.int32, device="cuda")
    k_new = qkv_h[1, :, :hkv].contiguous()
    v_new = qkv_h[2, :, :hkv].contiguous()
    # device-resident reference path: append on the device, relay step
    paged.append_slots(0, k_new.cuda(), v_new.cuda(), slots)
    ref = step(qkv_h[0].cuda())[0].clone()
    torch.cuda.synchronize()
    out_e = torch.empty((b, hq, 128), dtype=torch.bfloat16).pin_memory()
    step.step_host(qkv_h[0], k_new, v_new, slots, out_e)
    torch.cuda.synchronize()
    assert torch.equal(out_e, ref.cpu()), "step_host differs from the device path"
    out_g = torch.zeros((b, hq, 128), dtype=torch.bfloat16).pin_memory()
    # host_step_graph takes one (3, b, h, 128) buffer: h = hq = hkv only;
    # both the zero-copy graph (kernels read / write pinned host memory) and
    # the staged-copy graph
    if hq == hkv:
        qkv_eq = torch.stack([qkv_h[0], k_new, v_new]).pin_memory()
        for zc in (True, False):
            out_g.zero_()
            replay = step.host_step_graph(qkv_eq, slots, out_g, zero_copy=zc)
            replay()
            torch.cuda.synchronize()
            assert torch.equal(out_g, ref.cpu()), f"host_step_graph(zero_copy={zc}) differs"
    pairs = [(r, h) for r in range(b) for h in sorted({0, hkv - 1})]
    check_sampled_pairs(oracle, out_e.cuda().float(), step.lse, qkv_h[0].cuda(), sys_cache, paged, 0,
                        pairs, hq // hkv, f"e2e host step b={b} g={hq // hkv}")


@pytest.mark.parametrize("hq,hkv,bs", [(8, 8, 16), (16, 4, 32), (8, 2, 8)])
def test_fused_append_equals_separate_append(oracle, hq, hkv, bs):
    """rb_relay_attention with k_new / v_new / slot_mapping (the append fused
    into the context kernel) == rb_kv_append followed by the step, bitwise,
    with the new tokens landing at their slots; new K / V read from device
    memory and from pinned host memory."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    lens = [20, 1, 47, 16, 33]
    b = len(lens)
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, 300, lens, seed=hq + bs, block_size=bs)
    btc = bt.cpu()
    slots = torch.tensor([int(btc[r, (c - 1) // bs]) * bs + (c - 1) % bs for r, c in enumerate(lens)],
                         dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(1)
    k_new = torch.randn((b, hkv, 128), generator=g, device="cuda").to(torch.bfloat16)
    v_new = torch.randn((b, hkv, 128), generator=g, device="cuda").to(torch.bfloat16)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq, out_dtype=torch.float32)
    paged.append_slots(0, k_new, v_new, slots)
    ref = [t.clone() for t in step(q)]
    kpool, vpool = paged.k_pool.clone(), paged.v_pool.clone()
    for src in ("device", "host"):
        paged.k_pool.normal_()   # poison: the fused path must write the new rows itself
        paged.v_pool.copy_(vpool)
        paged.k_pool.copy_(kpool)
        for r, c in enumerate(lens):     # clear the new tokens' slots
            blk, off = int(btc[r, (c - 1) // bs]), (c - 1) % bs
            paged.k_pool[0, blk, :, off] = 0
            paged.v_pool[0, blk, :, off] = 0
        kn = k_new if src == "device" else k_new.cpu().pin_memory()
        vn = v_new if src == "device" else v_new.cpu().pin_memory()
        got = step(q, k_new=kn, v_new=vn, slot_mapping=slots)
        torch.cuda.synchronize()
        assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]), f"fused append ({src})"
        assert torch.equal(paged.k_pool, kpool) and torch.equal(paged.v_pool, vpool), f"pool ({src})"
    pairs = [(r, h) for r in range(b) for h in sorted({0, hkv - 1})]
    check_sampled_pairs(oracle, ref[0], ref[1], q, sys_cache, paged, 0, pairs, hq // hkv,
                        f"fused append hq={hq} hkv={hkv} bs={bs}")


def test_resplit_follows_growing_contexts(oracle):
    """RelayDecodeStep.resplit: the SM split recomputed for the batch's
    current context length (a serving loop's contexts grow); the step stays
    correct under the new split."""
    from paper_2402_14808_b200 import _lib, kernels
    from paper_2402_14808_b200.attention import RelayDecodeStep
    lens = [64] * 16
    q, sys_cache, paged, bt, cl = synth_paged_problem(16, 8, 8, 4096, lens, seed=9)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, 8, out_dtype=torch.float32)
    g0 = step.grid
    big = 16 * 60000   # as if the contexts had grown to 60k tokens each
    changed = step.resplit(big)
    assert changed == (step.grid != g0)
    assert step.grid == _lib.relay_sys_grid(16, 8, 8, 4096, big, kernels.sm_count())
    assert step.grid < g0          # longer contexts: fewer system CTAs
    assert not step.resplit(big)   # unchanged split: nothing to do
    out, lse = step(q)
    torch.cuda.synchronize()
    check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, 0, [(r, 0) for r in range(16)], 1,
                        "relay step after resplit")


@pytest.mark.parametrize("b,hq,hkv,s", [(64, 32, 8, 300), (40, 64, 8, 520), (48, 48, 8, 260)])
def test_gqa2_query_loaders_agree(oracle, b, hq, hkv, s):
    """Query rows of the 256-row GQA system kernel: by TMA from device memory
    (g divides 128), by the cp.async loader otherwise (g = 6 here), and from
    pinned host memory through the step's staging copy.  Host and device q
    must give the same step bitwise, and the oracle's result on sampled
    pairs (b=40, g=8: a partial last unit, rows past the batch zero-filled)."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    lens = [1 + (7 * r) % 90 for r in range(b)]
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b + s)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    assert step.plan["nq"] == 256, step.plan
    ref = step(q)[0].clone()
    lse_ref = step.lse.clone()
    qh = q.cpu().pin_memory()
    step._launch(qh, 3)
    torch.cuda.synchronize()
    assert torch.equal(step.out, ref), "host-q (cp.async) and device-q (TMA) steps differ"
    assert torch.equal(step.lse, lse_ref)
    pairs = [(r, h) for r in (0, b // 2, b - 1) for h in (0, hkv - 1)]
    check_sampled_pairs(oracle, ref.float(), lse_ref, q, sys_cache, paged, 0, pairs, hq // hkv,
                        f"gqa2 loaders b={b} g={hq // hkv}")


@pytest.mark.parametrize("b,hq,hkv,s", [(24, 8, 8, 300), (16, 32, 8, 700)])
def test_claim_order_does_not_change_results(oracle, b, hq, hkv, s):
    """RelayDecodeStep claims the context work longest request first when
    the lengths differ (req_order); the step must be bitwise the same as in
    request order, and equal the oracle."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    lens = [1 + (37 * r) % 300 for r in range(b)]
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b * 3 + s)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    assert step.req_order is not None
    order = step.req_order.cpu().tolist()
    assert sorted(order) == list(range(b))
    assert all(lens[order[i]] >= lens[order[i + 1]] for i in range(b - 1))
    out_o = step(q)[0].clone()
    lse_o = step.lse.clone()
    step.req_order = None
    out_n = step(q)[0].clone()
    assert torch.equal(out_o, out_n) and torch.equal(lse_o, step.lse)
    pairs = [(r, h) for r in (0, b // 2, b - 1) for h in (0, hkv - 1)]
    check_sampled_pairs(oracle, out_o.float(), lse_o, q, sys_cache, paged, 0, pairs, hq // hkv,
                        f"claim order b={b} g={hq // hkv}")


@pytest.mark.parametrize("b,hq,hkv,s", [(8, 12, 4, 300), (6, 32, 8, 700)])
def test_swap_ab_query_loaders(oracle, b, hq, hkv, s):
    """Query rows of the swap-AB system kernels: by TMA when g divides the
    unit's rows (g = 4 here), by the cp.async loader otherwise (g = 3); the
    step equals the oracle either way and host q (staged) equals device q."""
    from paper_2402_14808_b200.attention import RelayDecodeStep
    lens = [1 + (11 * r) % 70 for r in range(b)]
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, seed=b + s + hq)
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    assert step.plan["nq"] in (16, 32), step.plan
    ref = step(q)[0].clone()
    lse_ref = step.lse.clone()
    step._launch(q.cpu().pin_memory(), 3)
    torch.cuda.synchronize()
    assert torch.equal(step.out, ref) and torch.equal(step.lse, lse_ref)
    pairs = [(r, h) for r in (0, b - 1) for h in (0, hkv - 1)]
    check_sampled_pairs(oracle, ref.float(), lse_ref, q, sys_cache, paged, 0, pairs, hq // hkv,
                        f"swap-AB loaders b={b} g={hq // hkv}")
