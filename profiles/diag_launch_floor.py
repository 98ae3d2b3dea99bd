"""Fixed per-step cost of the harness and of each launch shape: CUDA-graph
replay of (a) a trivial elementwise kernel, (b) the system kernel on one tiny
tile (one CTA, ~200 KB smem), (c) the whole relay step at a tiny size, each
timed with events around the replay after the bench's L2 flush.  Diagnostics.

    python profiles/diag_launch_floor.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402


def timed(fn, flush, n=30):
    g = bench.graph_of(torch, fn)
    ts = []
    for _ in range(n):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[n // 2]


def main():
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    x = torch.zeros(1024, device=dev)
    print(f"trivial kernel          {timed(lambda: x.add_(1.0), flush):6.1f} us")
    q = torch.randn(1, 1, 128, device=dev).to(torch.bfloat16)
    sk = torch.randn(128, 1, 128, device=dev).to(torch.bfloat16)
    print(f"system kernel, 1 tile   {timed(lambda: kernels.system_attention(q, sk, sk, grid=1), flush):6.1f} us")
    for s in (128, 512):
        qq, relay, _, _, _ = bench.build(torch, s, list(range(2)), dev)
        print(f"relay step s={s:<5d} 2 heads {timed(lambda: relay(qq), flush):6.1f} us")
    print(f"no flush: trivial {timed(lambda: x.add_(1.0), lambda: None):6.1f} us")


if __name__ == "__main__":
    main()
