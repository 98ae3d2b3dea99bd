"""C3 (32-layer decode-attention stack, b=64, 32 heads, s=4096, c ~ U[64,768])
under SM-split and claim-order variants: graph-replayed stack, L2 flushed,
CUDA events (bench.py's timing).

    python profiles/diag_c3_stack.py [grid ...]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStack  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    import numpy as np
    lens = [int(x) for x in np.random.default_rng(1002).integers(64, 769, size=64)]
    q, sc, paged, bt, cl = bench.build_workload(torch, 64, 32, 32, 4096, lens, list(range(32)), dev,
                                                seed=77, layers=32)
    qs = q[None].expand(32, *q.shape).contiguous()
    grids = [int(x) for x in sys.argv[1:]] or [None]
    for grid in grids:
        for ordered in (True, False):
            st = RelayDecodeStack(sc, paged, bt, cl, hq=32, grid=grid)
            if not ordered:
                for s_ in st.steps:
                    s_.req_order = None
            g = bench.graph_of(torch, lambda: st(qs))
            ms = statistics.mean(bench.time_loop(torch, g.replay, 5, 3, flush))
            print(f"grid {grid} (plan {st.plan['grid']}, rr {st.plan['rr']}) ordered={ordered}: "
                  f"{ms * 1e3:.1f} us per stack", flush=True)
            del st, g


if __name__ == "__main__":
    main()
