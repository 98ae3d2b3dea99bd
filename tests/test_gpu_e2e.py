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
    # host_step_graph takes one (3, b, h, 128) buffer: h = hq = hkv only
    if hq == hkv:
        qkv_eq = torch.stack([qkv_h[0], k_new, v_new]).pin_memory()
        replay = step.host_step_graph(qkv_eq, slots, out_g)
        replay()
        torch.cuda.synchronize()
        assert torch.equal(out_g, ref.cpu()), "host_step_graph differs from the device path"
    pairs = [(r, h) for r in range(b) for h in sorted({0, hkv - 1})]
    check_sampled_pairs(oracle, out_e.cuda().float(), step.lse, qkv_h[0].cuda(), sys_cache, paged, 0,
                        pairs, hq // hkv, f"e2e host step b={b} g={hq // hkv}")
