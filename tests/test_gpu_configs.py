"""Full-size parity at the BASELINE.json configurations (one decode layer).

Each test builds the config's relay decode step at full size on the GPU
(seeded normal bf16 inputs resident in HBM), runs the product path
(RelayDecodeStep: tcgen05 system kernel || paged context kernel with the
relay fusion in its epilogue) and checks it against the float64 oracle on
sampled (request, KV-head group) pairs -- the oracle attends the new token
over the whole [system || context] sequence, which is what the relay output
and the fused LSE must equal (attention.py:203-243; eqs. 4-6).
The naive per-request kernel (`baseline_attention`, attention.py:266-296) is
compared at full size as a second, size-independent check.

  C2  Llama-30B attention, 52 heads, b=32, c=128, s=8192   (configs[1])
  C3  Llama-2-7B layer, 32 heads, b=64, s=4096, c~U[64,768] (configs[2])
  C4  Llama-3-8B GQA 32q/8kv, b=128, s=32768, c=512         (configs[3])
  C5  Llama-2-70B GQA 64q/8kv, b=256, s=65536, c=1024       (configs[4])
"""

import numpy as np
import pytest
import torch

from gpu_util import (assert_close, check_sampled_pairs, log_parity,
                      synth_paged_problem)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rb():
    from paper_2402_14808_b200 import _lib
    _lib.load()
    import paper_2402_14808_b200 as pkg
    return pkg


CONFIGS = {
    "C2": dict(b=32, hq=52, hkv=52, s=8192, lens=[128] * 32, seed=1001),
    "C3": dict(b=64, hq=32, hkv=32, s=4096,
               lens=[int(x) for x in np.random.default_rng(1002).integers(64, 769, size=64)],
               seed=1002),
    "C4": dict(b=128, hq=32, hkv=8, s=32768, lens=[512] * 128, seed=1003),
    "C5": dict(b=256, hq=64, hkv=8, s=65536, lens=[1024] * 256, seed=1004),
}


def _run_config(rb, oracle, name, expect_plan=None, naive=True):
    from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep
    cfg = CONFIGS[name]
    b, hq, hkv, s, lens = cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"], cfg["lens"]
    q, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, cfg["seed"])
    step = RelayDecodeStep(sys_cache, paged, bt, cl, hq)
    if expect_plan:
        for k, v in expect_plan.items():
            assert step.plan[k] == v, (name, step.plan)
    out, lse = [t.clone() for t in step(q)]
    out2, lse2 = step(q)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2), f"{name}: step not deterministic"
    g = hq // hkv
    rng = np.random.default_rng(cfg["seed"])
    reqs = sorted({0, b - 1, *[int(x) for x in rng.integers(0, b, size=2)]})
    heads = sorted({0, hkv - 1, int(rng.integers(0, hkv))})
    pairs = [(r, h) for r in reqs for h in heads]
    o_max, o_rel, l_max = check_sampled_pairs(oracle, out, lse, q, sys_cache, paged, 0, pairs, g,
                                              f"{name} relay vs oracle")
    rec = dict(config=name, plan=step.plan, grid=step.grid, pairs=len(pairs), o_max_abs=o_max,
               o_rel=o_rel, lse_max_abs=l_max)
    if naive:
        nout, nlse = NaiveDecodeStep(sys_cache, paged, bt, cl, hq)(q)
        torch.cuda.synchronize()
        n_max, n_rel = assert_close(out.float().cpu().numpy(), nout.float().cpu().numpy(),
                                    f"{name} relay vs naive kernel (all heads)")
        nl_max, _ = assert_close(lse.cpu().numpy(), nlse.cpu().numpy(), f"{name} lse vs naive",
                                 lse=True)
        rec.update(naive_o_max_abs=n_max, naive_o_rel=n_rel, naive_lse_max_abs=nl_max)
    log_parity(f"config {name}", kind="config", **rec)


def test_c2_full_size(rb, oracle):
    _run_config(rb, oracle, "C2", expect_plan={"nq": 32, "n_qt": 1})


def test_c3_one_layer_full_size(rb, oracle):
    _run_config(rb, oracle, "C3", expect_plan={"nq": 32, "n_qt": 2})


def test_c4_full_size(rb, oracle):
    # 512 query rows per KV head: 256-row units (two query tiles, sys_gqa2)
    _run_config(rb, oracle, "C4", expect_plan={"nq": 256, "n_qt": 2})


def test_c5_full_size(rb, oracle):
    # 2048 rows per KV head: 8 units of 256 rows per head, 2 CTAs per unit
    _run_config(rb, oracle, "C5", expect_plan={"nq": 256, "n_qt": 8, "grid": 128, "rr": 0})


def test_c3_32_layer_stack(rb, oracle):
    """configs[2] as stated: the 32-layer decode-attention stack (b=64, 32
    heads, s=4096, paged 16-token blocks, c ~ U[64, 768]) through
    RelayDecodeStack -- one relay step per layer over per-layer caches --
    deterministic, and against the oracle on sampled layers / pairs."""
    from paper_2402_14808_b200.attention import RelayDecodeStack
    cfg = CONFIGS["C3"]
    b, hq, hkv, s, lens = cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"], cfg["lens"]
    layers = 32
    q0, sys_cache, paged, bt, cl = synth_paged_problem(b, hq, hkv, s, lens, 3003, layers=layers)
    gen = torch.Generator(device="cuda").manual_seed(3004)
    q = torch.randn((layers, b, hq, 128), device="cuda", generator=gen).to(torch.bfloat16)
    stack = RelayDecodeStack(sys_cache, paged, bt, cl, hq)
    out, lse = [t.clone() for t in stack(q)]
    out2, lse2 = stack(q)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2), "stack not deterministic"
    rng = np.random.default_rng(3005)
    worst = [0.0, 0.0, 0.0]
    for layer in (0, 13, layers - 1):
        pairs = [(int(r), int(h)) for r, h in zip(rng.integers(0, b, size=3), rng.integers(0, hkv, size=3))]
        res = check_sampled_pairs(oracle, out[layer], lse[layer], q[layer], sys_cache, paged,
                                  layer, pairs, 1, f"C3 layer {layer}")
        worst = [max(a, b_) for a, b_ in zip(worst, res)]
    log_parity("config C3 (32-layer stack)", kind="config", config="C3x32", layers=layers,
               sampled_layers=[0, 13, layers - 1], o_max_abs=worst[0], o_rel=worst[1],
               lse_max_abs=worst[2])
