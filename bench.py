"""Relay decode-attention benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Metric: decode attention us/step (and HBM GB/s) vs system-prompt length at
B=32 -- the reference's `relayserve profile-attn` measurement
(/root/reference/pkg/src/relayserve/cli.py:320-357) on BASELINE.json
configs[1]: Llama-30B attention shape (52 heads, d=128), batch 32, context
128, system prompt swept 512..32k; the headline `value` is s=8192 (the top of
configs[1]'s sweep).  One step = one relay decode step of one layer: the
tcgen05 system kernel over the shared prefix + the paged context kernel with
the fused relay epilogue.  Inputs are synthetic (seeded normal bf16, one
generator per KV head), resident in HBM; L2 (126 MB) is flushed between timed
steps (write a 2x-L2 buffer, then read another so the write-back happens
outside the timed region).  `value` is the CUDA-graph replay of the step
(eager launches reported beside it); `e2e` the CUDA-graph replay of the
host-buffer step (pinned H2D + paged append + step + D2H).

The other BASELINE configs are timed in the same run under `configs`: C3
(the 32-layer Llama-2-7B decode-attention stack, b=64, s=4k, c ~ U[64,768],
one CUDA graph of 32 relay steps), C4 (Llama-3-8B GQA, b=128, s=32k, c=512),
C5 (Llama-2-70B GQA, b=256, s=64k, c=1k), each with its roofline
max(B_alg/BW, F_sys/P_tc).

N > 1 (torchrun): KV heads are sharded across ranks (52 -> 7,7,7,7,6,6,6,6 at
N=8; C4/C5: one KV head per rank at N=8); each rank runs the same step on its
heads, no collective in the timed region; step time = max over ranks (fixed
total work: "strong").  After timing, the sharded output is all-gathered
(NCCL) and compared bitwise with the unsharded step computed on rank 0.

--impl reference times the reference's own CPU implementation (the
unmodified relayserve modules compiled into oracle/_ref by oracle/build.py,
float64, all host cores via head-parallel processes) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, H, C, D = 32, 52, 128, 128
HEADLINE_S = 8192
SWEEP = (512, 1024, 2048, 4096, 8192, 16384, 32768)
BLOCK = 16
METRIC = "decode attention µs/step & HBM GB/s vs sys-prompt length (B=32), 1/2/4/8 B200"
# BASELINE.json configs[3], configs[4] (one decode layer each)
OTHER = {
    "C3": dict(b=64, hq=32, hkv=32, s=4096, c="U[64,768]", layers=32,
               label="C3 Llama-2-7B decode-attention stack (configs[2]): 32 layers, b=64, H=32, "
                     "s=4096, paged 16, c ~ U[64,768] (seeded)"),
    "C4": dict(b=128, hq=32, hkv=8, s=32768, c=512,
               label="C4 Llama-3-8B GQA (configs[3]): b=128, 32q/8kv, s=32768, c=512"),
    "C5": dict(b=256, hq=64, hkv=8, s=65536, c=1024,
               label="C5 Llama-2-70B GQA (configs[4]): b=256, 64q/8kv, s=65536, c=1024"),
}
PARITY_HEADS = (0, 17, 34, 51)   # KV heads the CPU reference sample and parity check use


def workload_label(s):
    """config.workload of both arms (identical strings)."""
    return (f"C2 Llama-30B attention shape (configs[1]): b={B}, H={H}, d={D}, c={C}, s={s}, "
            f"paged block {BLOCK}")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--s", type=int, default=HEADLINE_S)
    p.add_argument("--sweep", type=str, default=",".join(map(str, SWEEP)))
    p.add_argument("--configs", type=str, default="C3,C4,C5")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU sampling")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cpu():
    model = platform.processor() or "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"lscpu_model": model, "logical_cpus": os.cpu_count()}


# ------------------------------------------------------------ measurement

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        loaded = [x for x in sm if smax and x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def make_flush(torch, device):
    """L2 flush between timed steps: write a 2x-L2 buffer, then read a second
    2x-L2 buffer.  The read evicts the written (dirty) lines, so their
    write-back to HBM happens here, outside the timed region, and the timed
    step starts with an L2 that holds none of its inputs."""
    l2 = torch.cuda.get_device_properties(device).L2_cache_size
    n = max(2 * l2, 256 << 20)
    wbuf = torch.empty(n, dtype=torch.uint8, device=device)
    rbuf = torch.ones(n // 4, dtype=torch.float32, device=device)
    sink = torch.empty((), dtype=torch.float32, device=device)

    def flush():
        wbuf.zero_()
        torch.amax(rbuf, dim=0, out=sink)
    return flush


def time_loop(torch, fn, steps, warmup, flush, barrier=None):
    """W warm-up steps, then exactly `steps` timed steps; per-step CUDA events
    on the launching (current) stream; L2 flushed before every step outside
    the events.  Returns per-step milliseconds."""
    for _ in range(warmup):
        flush()
        fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for a, b in ev:
        flush()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return [a.elapsed_time(b) for a, b in ev]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1647.2)),
                float(p.get("bf16_tflops_sustained", 1392.3)), "measured")
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def ncu_traffic(kernels, s):
    """dram bytes per step of `kernels` (summed) at system length s from the
    committed ncu summary (profiles/ncu_summary.json), if every one of them
    has an entry for this config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            data = json.load(f)
        return sum(data["kernels"][k][str(s)]["dram_bytes"] for k in kernels)
    except Exception:
        return None


# ---------------------------------------------------------------- workload

def build_workload(torch, b, hq, hkv, s, lens, kv_heads, device, seed=1234, layers=1):
    """Seeded synthetic decode workload holding the given global KV heads
    (and their g query heads): one generator per (layer, KV head), so a
    sharded run holds exactly the unsharded run's data for its heads.
    Returns (q, SystemKvCache, PagedKvCache, block_table, ctx_lens)."""
    from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache
    g = hq // hkv
    nh = len(kv_heads)
    gen = torch.Generator(device=device)
    nblk = sum(-(-c // BLOCK) for c in lens)
    paged = PagedKvCache(layers, nh, nblk, BLOCK, device=device)
    keys, values = [], []
    q = torch.empty((b, nh * g, D), dtype=torch.bfloat16, device=device)
    for layer in range(layers):
        sk = torch.empty((nh, s, D), dtype=torch.bfloat16, device=device)
        sv = torch.empty_like(sk)
        for i, hg in enumerate(kv_heads):
            gen.manual_seed((seed * 1000003 + hg) * 131 + layer)
            sk[i] = torch.randn((s, D), generator=gen, device=device)
            sv[i] = torch.randn((s, D), generator=gen, device=device)
            paged.k_pool[layer, :, i] = torch.randn((nblk, BLOCK, D), generator=gen, device=device)
            paged.v_pool[layer, :, i] = torch.randn((nblk, BLOCK, D), generator=gen, device=device)
            if layer == 0:
                q[:, i * g:(i + 1) * g] = torch.randn((b, g, D), generator=gen, device=device)
        keys.append(sk)
        values.append(sv)
    # shuffled physical blocks, as a real paged allocator would hand out
    paged.allocator.shuffle(seed)
    for r, c in enumerate(lens):
        paged.register(r)
        paged.extend(r, c)
    ids = list(range(b))
    return q, SystemKvCache(keys, values), paged, paged.block_table(ids), paged.context_lens(ids)


def graph_of(torch, fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fn()
    return graph


# ----------------------------------------------------------- CPU baselines

def _ref_modules():
    """The reference compiled in oracle/_ref ("reference") else the port."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "relayserve")):
        sys.path.insert(0, ref_dir)
        try:
            import relayserve.attention as att
            return att, "reference"
        except Exception:
            pass
    from oracle import relay_oracle
    return relay_oracle, "port"


_CPU = {}


def _cpu_data(s, nh, seed=7):
    import numpy as np
    rng = np.random.default_rng(seed)
    sk = rng.standard_normal((s, nh, D)); sv = rng.standard_normal((s, nh, D))
    ck = [rng.standard_normal((C, nh, D)) for _ in range(B)]
    cv = [rng.standard_normal((C, nh, D)) for _ in range(B)]
    q = rng.standard_normal((B, 1, nh, D))
    return q, sk, sv, ck, cv


def _cpu_worker(args):
    lo, hi = args
    att = _CPU["att"]
    q, sk, sv, ck, cv = _CPU["data"]
    t0 = time.perf_counter()
    att.relay_attention(q[:, :, lo:hi], sk[:, lo:hi], sv[:, lo:hi],
                        [x[:, lo:hi] for x in ck], [x[:, lo:hi] for x in cv])
    return time.perf_counter() - t0


def cpu_leg(torch, q, sys_cache, paged, out, lse, budget):
    """cpu_baseline of the N=1 line, on the GPU run's own inputs: the
    reference relay step (oracle/_ref, float64, 1 core) over the sampled KV
    heads, best-of-N within `budget` seconds, extrapolated linearly in heads
    (heads are independent and identical work, attention.py:122-133) -- and,
    on the same sample, the GPU step's output / fused LSE against the float64
    oracle (the checker; parity of the bench line)."""
    import numpy as np
    from oracle import relay_oracle as orc
    heads = [h for h in PARITY_HEADS if h < sys_cache.kv_heads]
    qn = q.float().cpu().numpy()[:, None][:, :, heads].astype(np.float64)
    sk = sys_cache.keys[0].float().cpu().numpy()[heads].transpose(1, 0, 2).astype(np.float64)
    sv = sys_cache.values[0].float().cpu().numpy()[heads].transpose(1, 0, 2).astype(np.float64)
    ck, cv = [], []
    for r in range(q.shape[0]):
        k_r, v_r = paged.gather(r, 0)
        ck.append(k_r.float().cpu().numpy()[:, heads].astype(np.float64))
        cv.append(v_r.float().cpu().numpy()[:, heads].astype(np.float64))
    ref_o, ref_l = orc.relay_attention(qn, sk, sv, ck, cv, return_lse=True)
    got_o = out.float().cpu().numpy()[:, heads]
    got_l = lse.float().cpu().numpy()[:, heads]
    d = got_o - ref_o[:, 0]
    parity = {"o_max_abs": float(np.abs(d).max()),
              "o_rel": float(np.linalg.norm(d) / np.linalg.norm(ref_o)),
              "lse_max_abs": float(np.abs(got_l - ref_l[:, 0]).max()),
              "heads": heads, "rows": int(q.shape[0]),
              "oracle": "float64 C restatement of the reference (oracle/relay_oracle), "
                        "same bf16 inputs",
              "tolerance": {"o_max_abs": 1.5e-2, "o_rel": 5e-3, "lse_max_abs": 1e-3}}
    att, kind = _ref_modules()
    best, reps, t0 = float("inf"), 0, time.perf_counter()
    while reps < 5 and (reps < 1 or time.perf_counter() - t0 < budget):
        t1 = time.perf_counter()
        att.relay_attention(qn, sk, sv, ck, cv)
        best = min(best, time.perf_counter() - t1)
        reps += 1
    nh = len(heads)
    cpu = {"value": best * 1e6 * H / nh, "unit": "µs/step", "cores": 1, "kind": kind,
           "sample": (f"relay_attention on the GPU run's own bf16 inputs (b={B}, "
                      f"s={sys_cache.system_len}, c={C}, d={D}), {nh} of {H} heads, best of "
                      f"{reps} on 1 core, float64, extrapolated x{H / nh:g} to all heads"),
           "host": host_cpu()}
    return cpu, parity


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp
    att, kind = _ref_modules()
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, H))
    _CPU["att"], _CPU["data"] = att, _cpu_data(args.s, H)
    bounds = [(H * i // procs, H * (i + 1) // procs) for i in range(procs)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_worker, bounds)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, bounds)
            times.append(time.perf_counter() - t0)
    us = statistics.mean(times) * 1e6
    sample = (f"full workload per step: relay_attention b={B}, {H} heads, s={args.s}, c={C}, "
              f"d={D}, float64, heads split over {procs} processes")
    line = {"metric": METRIC, "value": us, "unit": "µs/step", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": us / 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded normal)",
            "config": {"workload": workload_label(args.s), "global_batch": B, "seq_len": args.s,
                       "parallelism": f"host processes x{procs}"},
            "cpu_baseline": {"value": us, "unit": "µs/step", "cores": procs, "kind": kind,
                             "sample": sample, "host": host_cpu()},
            "e2e": {"value": us, "unit": "µs/step", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- GPU arm

def run_b200(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        args.gpus = world
    # BENCH_SAME_GPU=1 (testing only): every rank on cuda:0 with gloo, to
    # exercise the sharded path on a single-GPU box.
    same_gpu = os.environ.get("BENCH_SAME_GPU") == "1"
    local = 0 if same_gpu else local
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    barrier = None
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
        barrier = dist.barrier
    from paper_2402_14808_b200 import _lib, kernels, sharding
    from paper_2402_14808_b200.attention import NaiveDecodeStep, RelayDecodeStep
    from paper_2402_14808_b200.costmodel import DecodeShape
    _lib.load()
    ka, kb, _, _ = sharding.local_heads(H, H, world, rank)
    heads = list(range(ka, kb))
    flush = make_flush(torch, device)
    hbm, tc_burst, tc_sus, peak_kind = measured_peaks()

    def timed(fn, steps=None):
        return time_loop(torch, fn, steps or args.steps, args.warmup, flush, barrier)

    def c2_step(s, full=False):
        q, sc, paged, bt, cl = build_workload(torch, B, H, H, s, [C] * B, heads, device)
        relay = RelayDecodeStep(sc, paged, bt, cl, hq=len(heads))
        res = {"plan": relay.plan, "sys_grid": relay.grid}
        gr = graph_of(torch, lambda: relay(q))
        res["graph_ms"] = statistics.mean(timed(gr.replay))
        naive = NaiveDecodeStep(sc, paged, bt, cl, hq=len(heads))
        res["naive_ms"] = statistics.mean(time_loop(torch, lambda: naive(q), max(3, args.steps // 5),
                                                    2, flush, barrier))
        out_r, lse_r = [t.clone() for t in relay(q)]
        out_n = naive(q)[0]
        torch.cuda.synchronize()
        res["relay_vs_naive_max_abs"] = float((out_r.float() - out_n.float()).abs().max())
        if full:
            res["eager_ms"] = statistics.mean(timed(lambda: relay(q)))
            # each kernel alone on every SM (the step runs them concurrently
            # on a byte-proportional SM split)
            alone = RelayDecodeStep(sc, paged, bt, cl, len(heads), grid=kernels.sm_count(device))
            res["sys_ms"] = statistics.mean(timed(lambda: alone.system(q)))
            res["ctx_ms"] = statistics.mean(timed(lambda: alone.context(q)))
            del alone
            res.update(e2e_stats(q, relay, bt))
            # e2e wrote its new tokens into the pool: the parity leg re-runs
            # the step on the cache as it is now
            out_p, lse_p = [t.clone() for t in relay(q)]
            res["objs"] = (q, sc, paged, out_p, lse_p)
        del relay, naive, gr
        return res

    def e2e_stats(q, relay, bt):
        """Public-API decode step with host buffers: this step's q / new-token
        k / v cross from pinned memory, are appended and attended, and the
        output crosses back -- all inside the events (RelayDecodeStep.
        host_step_graph: one CUDA graph of the zero-copy step, whose kernels
        read the inputs from / write the output to pinned host memory;
        `step_host` is the eager copy-based equivalent)."""
        nh = q.shape[1]
        g = torch.Generator().manual_seed(99)
        qkv_h = torch.randn((3, B, nh, D), generator=g).to(torch.bfloat16).pin_memory()
        out_h = torch.empty((B, nh, D), dtype=torch.bfloat16).pin_memory()
        # the step's new token overwrites slot c-1 of each request (context
        # length stays c, so every timed step does identical work)
        btc = bt.cpu()
        slots = torch.tensor([int(btc[r, (C - 1) // BLOCK]) * BLOCK + (C - 1) % BLOCK
                              for r in range(B)], dtype=torch.int32, device=device)
        eager = lambda: relay.step_host(qkv_h[0], qkv_h[1], qkv_h[2], slots, out_h)  # noqa: E731
        ms_eager = timed(eager)
        replay = relay.host_step_graph(qkv_h, slots, out_h)
        ms = timed(replay)
        return {"e2e_graph_ms": statistics.mean(ms), "e2e_eager_ms": statistics.mean(ms_eager),
                "h2d": qkv_h.numel() * 2, "d2h": out_h.numel() * 2}

    def other_lens(cfg):
        if isinstance(cfg["c"], int):
            return [cfg["c"]] * cfg["b"]
        import numpy as np
        return [int(x) for x in np.random.default_rng(1002).integers(64, 769, size=cfg["b"])]

    def other_config(name):
        from paper_2402_14808_b200.attention import RelayDecodeStack
        cfg = OTHER[name]
        b, hq, hkv, s = cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"]
        layers = cfg.get("layers", 1)
        lens = other_lens(cfg)
        a, bb, _, _ = sharding.local_heads(hkv, hq, world, rank)
        kvh = list(range(a, bb))
        g = hq // hkv
        q, sc, paged, bt, cl = build_workload(torch, b, hq, hkv, s, lens, kvh, device, seed=77,
                                              layers=layers)
        if layers > 1:
            qs = q[None].expand(layers, *q.shape).contiguous()
            step = RelayDecodeStack(sc, paged, bt, cl, hq=len(kvh) * g)
            fn = lambda: step(qs)  # noqa: E731
        else:
            step = RelayDecodeStep(sc, paged, bt, cl, hq=len(kvh) * g)
            fn = lambda: step(q)  # noqa: E731
        gr = graph_of(torch, fn)
        ms = statistics.mean(timed(gr.replay, max(5, args.steps // 2)))
        shp = DecodeShape(b, len(kvh) * g, len(kvh), s, sum(lens))
        res = {"label": cfg["label"], "kv_heads_per_rank": len(kvh), "layers": layers,
               "plan": step.plan, "sys_grid": step.grid, "ms": ms,
               "bytes_alg_per_rank": layers * shp.bytes_alg,
               "flops_sys_per_rank": layers * shp.flops_sys, "launches_per_step": 2 * layers}
        del step, gr, q, sc, paged
        torch.cuda.empty_cache()
        return res

    clocks = ClockSampler(local)
    t_wall = time.perf_counter()
    head = c2_step(args.s, full=True)
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline:
        q, sc, paged, out_r, lse_r = head["objs"]
        cpu, parity = cpu_leg(torch, q, sc, paged, out_r, lse_r, args.cpu_budget)
    head.pop("objs")
    torch.cuda.empty_cache()
    sweep = []
    for s in [int(x) for x in args.sweep.split(",") if x.strip()]:
        st = head if s == args.s else c2_step(s)
        torch.cuda.empty_cache()
        shp = DecodeShape(B, len(heads), len(heads), s, B * C)
        sweep.append({"s": s, "us_per_step": st["graph_ms"] * 1e3,
                      "naive_us_per_step": st["naive_ms"] * 1e3,
                      "bytes_alg_per_rank": shp.bytes_alg,
                      "relay_vs_naive_max_abs": st["relay_vs_naive_max_abs"]})
    others = {name: other_config(name) for name in [x for x in args.configs.split(",") if x]}
    clk = clocks.stop()
    wall = time.perf_counter() - t_wall

    def maxr(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if same_gpu else device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # every collective before rank 0 alone builds the line (the others exit)
    ms = maxr(head["graph_ms"])
    sys_ms, ctx_ms = maxr(head["sys_ms"]), maxr(head["ctx_ms"])
    e2e_ms = maxr(head["e2e_graph_ms"])
    eager_ms, naive_ms = maxr(head["eager_ms"]), maxr(head["naive_ms"])
    e2e_eager_ms = maxr(head["e2e_eager_ms"])
    for row in sweep:
        row["us_per_step"] = maxr(row["us_per_step"])
        row["naive_us_per_step"] = maxr(row["naive_us_per_step"])
        full = DecodeShape(B, H, H, row["s"], B * C)
        t = row["us_per_step"] * 1e-6
        row["hbm_gbs"] = full.bytes_alg / t / 1e9           # whole job over the slowest rank
        row["frac_of_hbm_roofline"] = full.bytes_alg / (world * hbm * 1e9) / t
        row["naive_bytes_over_relay"] = full.bytes_naive / full.bytes_alg
    for name, r in others.items():
        r["us_per_step"] = maxr(r["ms"]) * 1e3
        cfg = OTHER[name]
        L = cfg.get("layers", 1)
        full = DecodeShape(cfg["b"], cfg["hq"], cfg["hkv"], cfg["s"], sum(other_lens(cfg)))
        t = r["us_per_step"] * 1e-6
        t_hbm = L * full.bytes_alg / (world * hbm * 1e9)
        t_tc = L * full.flops_sys / (world * tc_sus * 1e12)
        r.update({"bytes_alg": L * full.bytes_alg, "flops_sys": L * full.flops_sys,
                  "roofline_us": max(t_hbm, t_tc) * 1e6, "frac_of_roofline": max(t_hbm, t_tc) / t,
                  "bound": "tensor" if t_tc > t_hbm else "hbm",
                  "sys_tflops": L * full.flops_sys / t / 1e12, "tokens_per_s": cfg["b"] / t,
                  "peaks": f"HBM {hbm} GB/s, bf16 {tc_sus} TF/s sustained ({peak_kind}), x{world} GPUs"})
        r.pop("ms")

    # end-to-end check of the sharded path: all-gather the per-rank outputs
    # and compare bitwise with the unsharded step (rank 0).  Both sides cut
    # every system unit at the same key tiles (k CTAs per unit), the
    # condition for bitwise equality (tests/test_gpu_sharding.py).
    sharded_equal = None
    if world > 1:
        s_chk, k_unit = 1024, 2
        q, sc, paged, bt, cl = build_workload(torch, B, H, H, s_chk, [C] * B, heads, device)
        n_units = _lib.sys_plan(B, len(heads), len(heads), s_chk, 148)[0]["n_units"]
        out, _ = RelayDecodeStep(sc, paged, bt, cl, len(heads), grid=k_unit * n_units)(q)
        torch.cuda.synchronize()
        full = sharding.gather_heads(out.cpu() if same_gpu else out, H, H)
        if rank == 0:
            q, sc, paged, bt, cl = build_workload(torch, B, H, H, s_chk, [C] * B, list(range(H)),
                                                  device)
            n_all = _lib.sys_plan(B, H, H, s_chk, 148)[0]["n_units"]
            ref, _ = RelayDecodeStep(sc, paged, bt, cl, H, grid=k_unit * n_all)(q)
            torch.cuda.synchronize()
            sharded_equal = bool(torch.equal(full.to(ref.device), ref))
        del q, sc, paged

    if rank != 0:
        dist.destroy_process_group()
        return 0

    shape = DecodeShape(B, H, H, args.s, B * C)
    step_bytes_local = DecodeShape(B, len(heads), len(heads), args.s, B * C).bytes_alg
    sys_bytes_local = 2 * 2 * len(heads) * D * args.s + 2 * B * len(heads) * D
    # roofline of the step: the system and context kernels stream
    # concurrently on disjoint SMs, so the bound is the whole step's
    # algorithmic bytes (this rank's share) over the step time
    achieved = step_bytes_local / (ms * 1e-3) / 1e9
    value_us = ms * 1e3
    line = {
        "metric": METRIC, "value": value_us, "unit": "µs/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded normal), inputs resident in HBM",
        "config": {"workload": workload_label(args.s),
                   "global_batch": B, "seq_len": args.s,
                   "parallelism": f"kv-head-shard{world}" if world > 1 else "single-gpu",
                   "l2": "flushed between timed steps: write a 2x-L2 buffer, then read another 2x-L2 buffer (evicts inputs, write-back outside the timed region)",
                   "timing": "value = CUDA-graph replay of the 2-kernel step (the serving path); eager launches in eager_us_per_step",
                   "sys_sm_split": head["sys_grid"]},
        "tokens_per_s": B / (ms * 1e-3),
        "hbm_gbs": shape.bytes_alg / (ms * 1e-3) / 1e9,
        "frac_of_hbm_roofline": shape.bytes_alg / (world * hbm * 1e9) / (ms * 1e-3),
        "bytes_alg": shape.bytes_alg, "bytes_naive": shape.bytes_naive,
        "eager_us_per_step": eager_ms * 1e3,
        "naive_us_per_step": naive_ms * 1e3,
        "sys_kernel_alone_us": sys_ms * 1e3, "ctx_kernel_alone_us": ctx_ms * 1e3,
        "sys_kernel_alone_gbs": sys_bytes_local / (sys_ms * 1e-3) / 1e9,
        "ctx_kernel_alone_gbs": (step_bytes_local - sys_bytes_local) / (ctx_ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm",
                     "kernel": "relay step: sys_attn_sm100_kernel || ctx_cta_kernel (concurrent, relay fusion in-kernel)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "traffic": ncu_traffic(("sys_attn_sm100_kernel", "ctx_cta_kernel"), args.s),
                     "algorithmic_bytes_per_launch": step_bytes_local},
        "e2e": {"value": e2e_ms * 1e3, "unit": "µs/step", "h2d_bytes_per_step": head["h2d"],
                "d2h_bytes_per_step": head["d2h"],
                "path": "RelayDecodeStep.host_step_graph (CUDA graph, zero-copy): rb_relay_attention "
                        "stages q from the pinned host buffer into device memory (q_stage_kernel, "
                        "PDL-overlapped with the system kernel's K/V prefetch), reads the new tokens' "
                        "K/V from pinned memory and appends them inside the context kernel, runs "
                        "system || context with the fusion in-kernel and writes the output rows into "
                        "pinned host memory",
                "eager_us": e2e_eager_ms * 1e3, "eager_path": "step_host: H2D copies, rb_kv_append, "
                "the relay step, D2H copy", "launches_per_step": 3},
        "gpu_launches": 2 * args.steps,
        "relay_vs_naive_max_abs": head["relay_vs_naive_max_abs"],
        "sys_plan": head["plan"],
        "sweep": sweep, "configs": others, "clocks": clk, "wall_s": wall,
    }
    if parity is not None:
        line["parity"] = parity
    if sharded_equal is not None:
        line["sharded_equals_unsharded_bitwise"] = sharded_equal
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
