"""Measure the relay decode step on every BASELINE.json config (one layer,
one GPU, the whole KV-head range), beside the naive per-request kernel.

    python profiles/bench_configs.py [--steps K] [--configs c1,c2,c3,c4,c5]

The headline contract line is bench.py (configs[1] = C2); this script gives
the per-config table DESIGN.md quotes.  Same timing rules as bench.py: L2
flushed between steps, CUDA events on the launching stream, warm-up first.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402
from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep  # noqa: E402
from paper_2402_14808_b200.costmodel import DecodeShape  # noqa: E402
from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache  # noqa: E402

CONFIGS = {
    # name: (b, hq, hkv, s, ctx lengths spec)
    "c1": dict(b=4, hq=32, hkv=32, s=512, ctx="64"),
    "c2": dict(b=32, hq=52, hkv=52, s=8192, ctx="128"),
    "c3": dict(b=64, hq=32, hkv=32, s=4096, ctx="U64-768"),
    "c4": dict(b=128, hq=32, hkv=8, s=32768, ctx="512"),
    "c5": dict(b=256, hq=64, hkv=8, s=65536, ctx="1024"),
}


def ctx_lens(spec, b, seed=5):
    if spec.startswith("U"):
        lo, hi = (int(x) for x in spec[1:].split("-"))
        g = torch.Generator().manual_seed(seed)
        return torch.randint(lo, hi + 1, (b,), generator=g).tolist()
    return [int(spec)] * b


def build(cfg, device, seed=7):
    b, hq, hkv, s = cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"]
    lens = ctx_lens(cfg["ctx"], b)
    g = torch.Generator(device=device).manual_seed(seed)
    sys_cache = SystemKvCache.random(1, hkv, s, device=device, generator=g)
    nblk = sum(-(-c // 16) for c in lens)
    paged = PagedKvCache(1, hkv, nblk, 16, device=device)
    paged.k_pool.normal_(generator=g)
    paged.v_pool.normal_(generator=g)
    paged.allocator.shuffle(seed)
    for r, c in enumerate(lens):
        paged.register(r)
        paged.extend(r, c)
    ids = list(range(b))
    bt, cl = paged.block_table(ids), paged.context_lens(ids)
    q = torch.randn((b, hq, 128), device=device, generator=g).to(torch.bfloat16)
    return q, sys_cache, paged, bt, cl, lens


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--naive", action="store_true", help="also time the naive kernel")
    ap.add_argument("--grids", default="", help="diagnostics: also time these system-kernel SM splits")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    hbm, _, tc, _ = bench.measured_peaks()
    rows = []
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        q, sys_cache, paged, bt, cl, lens = build(cfg, dev)
        relay = RelayDecodeStep(sys_cache, paged, bt, cl, cfg["hq"])
        gr = bench.graph_of(torch, lambda: relay(q))
        ms = statistics.mean(bench.time_loop(torch, gr.replay, args.steps, args.warmup, flush))
        # the system kernel alone on every SM (the step shares SMs with the context kernel)
        alone = RelayDecodeStep(sys_cache, paged, bt, cl, cfg["hq"], grid=kernels.sm_count(dev))
        gs = bench.graph_of(torch, lambda: alone.system(q))
        sys_ms = statistics.mean(bench.time_loop(torch, gs.replay, args.steps, args.warmup, flush))
        shp = DecodeShape(cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"], sum(lens))
        t_star = shp.roofline_s(hbm * 1e9, tc * 1e12)
        row = {"config": name, **cfg, "ctx_total": sum(lens), "us_per_step": ms * 1e3,
               "sys_kernel_us": sys_ms * 1e3, "bytes_alg": shp.bytes_alg,
               "flops_sys": shp.flops_sys, "hbm_gbs": shp.bytes_alg / (ms * 1e-3) / 1e9,
               "roofline_us": t_star * 1e6, "frac_of_roofline": t_star / (ms * 1e-3),
               "bound": "tensor" if shp.flops_sys / (tc * 1e12) > shp.bytes_alg / (hbm * 1e9) else "hbm",
               "plan": relay.plan, "sys_alone_plan": alone.plan}
        if args.grids:
            sweep = {}
            for gsel in (int(x) for x in args.grids.split(",")):
                other = RelayDecodeStep(sys_cache, paged, bt, cl, cfg["hq"], grid=gsel)
                go = bench.graph_of(torch, lambda: other(q))
                sweep[gsel] = round(statistics.mean(
                    bench.time_loop(torch, go.replay, args.steps, args.warmup, flush)) * 1e3, 1)
                del other, go
            row["split_sweep_us"] = sweep
        if args.naive:
            naive = NaiveDecodeStep(sys_cache, paged, bt, cl, cfg["hq"])
            row["naive_us_per_step"] = statistics.mean(
                bench.time_loop(torch, lambda: naive(q), max(3, args.steps // 4), 1, flush)) * 1e3
        print(json.dumps(row), flush=True)
        rows.append(row)
        del q, sys_cache, paged, relay, alone, gr, gs
        torch.cuda.empty_cache()
    out = os.path.join(ROOT, "gpurun_out", "bench_configs.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
