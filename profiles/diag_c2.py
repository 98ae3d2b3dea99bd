"""C2 relay step (b=32, 52 heads, c=128) at several system lengths: graph-
replayed step time after the bench's L2 flush (median of 30), the production
SM split, plus the system kernel alone on every SM.  Compare library variants
with RB_LIB=<path>.  Diagnostics.

    python profiles/diag_c2.py [s1,s2,...]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402


def timed(fn, flush, n=30):
    g = bench.graph_of(torch, fn)
    return statistics.median(bench.time_loop(torch, g.replay, n, 3, flush)) * 1e3


def main():
    ss = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [512, 2048, 8192, 32768]
    b, h, c = 32, 52, 128
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    print(f"lib {os.environ.get('RB_LIB', 'default')}")
    for s in ss:
        q, sc, paged, bt, cl = bench.build_workload(torch, b, h, h, s, [c] * b, list(range(h)), dev)
        step = RelayDecodeStep(sc, paged, bt, cl, h)
        t = timed(lambda: step(q), flush)
        alone = RelayDecodeStep(sc, paged, bt, cl, h, grid=kernels.sm_count(dev))
        ts = timed(lambda: alone.system(q), flush)
        byt = 2 * 2 * h * 128 * (s + b * c) + 2 * b * h * 128
        print(f"s={s:6d} grid {step.grid:3d}: step {t:7.1f} us ({byt / t / 1e3:5.0f} GB/s)   "
              f"system kernel alone {ts:6.1f} us")
        del q, sc, paged, step, alone


if __name__ == "__main__":
    main()
