"""Sweep the system-kernel CTA count of the concurrent relay step (the SM
split between the system and context kernels) on the C2 workload.

    python profiles/sweep_split.py [s ...]

Per s: the split rb_relay_sys_grid picks, then graph-replayed step times
(L2 flushed between steps, CUDA events, min of 3 x 20 steps) for a range of
system grids.  Diagnostics only.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402


def time_step(fn, flush, steps=20):
    g = bench.graph_of(torch, fn)
    best = float("inf")
    for _ in range(3):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for e0, e1 in ev:
            flush()
            e0.record()
            g.replay()
            e1.record()
        torch.cuda.synchronize()
        best = min(best, sorted(e0.elapsed_time(e1) for e0, e1 in ev)[steps // 2] * 1e3)
    return best


def main():
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    sms = kernels.sm_count(dev)
    for s in [int(x) for x in (sys.argv[1:] or ["2048", "8192", "32768"])]:
        q, sc, paged, bt, cl = bench.build_workload(torch, bench.B, bench.H, bench.H, s,
                                                    [bench.C] * bench.B, list(range(bench.H)), dev)
        auto = _lib.relay_sys_grid(bench.B, bench.H, bench.H, s, bench.B * bench.C, sms)
        res = []
        grids = os.environ.get("SWEEP_GRIDS", "10,20,30,40,50,60,70,80,90,100,110,120,148")
        for g in sorted({auto} | {int(x) for x in grids.split(",")}):
            step = RelayDecodeStep(sc, paged, bt, cl, bench.H, grid=g)
            res.append((g, time_step(lambda: step(q), flush)))
        print(f"s={s} auto grid {auto}: " + ", ".join(f"{g}:{t:.1f}" for g, t in res), flush=True)


if __name__ == "__main__":
    main()
