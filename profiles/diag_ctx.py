"""Context kernel alone at C2 (b=32, 52 heads, c=128, paged 16): plain
context attention (rb_context_attention) and the relay step's context phase
(phases=2, system units already published), L2 flushed, CUDA events.
Diagnostics (ncu target: -k regex:ctx_cta).

    python profiles/diag_ctx.py [b h c reps]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402


def main():
    b, h, c, reps = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 52, 128, 20)))
    dev = torch.device("cuda", 0)
    q, sc, paged, bt, cl = bench.build_workload(torch, b, h, h, 1024, [c] * b, list(range(h)), dev)
    flush = bench.make_flush(torch, dev)
    step = RelayDecodeStep(sc, paged, bt, cl, h, grid=kernels.sm_count(dev))
    step.system(q)
    plain = lambda: kernels.context_attention(  # noqa: E731
        q, step.q_start, paged.k_pool[0], paged.v_pool[0], cl, max_rows=1, hkv=h, block_table=bt,
        block_size=16, strides=paged.strides(), out=step.out, lse_out=step.lse)
    byt = 2 * 2 * h * 128 * b * c
    for name, fn in (("plain", plain), ("relay ctx phase", lambda: step.context(q))):
        ms = bench.time_loop(torch, fn, reps, 3, flush)
        t = statistics.mean(ms) * 1e-3
        print(f"{name}: {t * 1e6:.1f} us  {byt / t / 1e9:.0f} GB/s of {byt / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
