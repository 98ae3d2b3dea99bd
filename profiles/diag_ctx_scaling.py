"""Context kernel alone vs context size: fixed cost + streaming rate.

Plain context attention (rb_context_attention, no relay) over paged KV,
b requests x h KV heads (g = 1), context c swept; CUDA-graph replay after
the bench's L2 flush, CUDA events.  Beside it: the harness floor (a trivial
kernel) and a torch streaming read (torch.sum) of the same byte count --
the achievable event-timed time for that many HBM bytes.  Diagnostics.

    python profiles/diag_ctx_scaling.py [b h c1,c2,...]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402


def timed(fn, flush, n=20):
    g = bench.graph_of(torch, fn)
    ms = bench.time_loop(torch, g.replay, n, 3, flush)
    return statistics.median(ms) * 1e3


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 52
    cs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [64, 128, 256, 512, 1024]
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    x = torch.zeros(1024, device=dev)
    print(f"floor: trivial kernel {timed(lambda: x.add_(1.0), flush):.1f} us")
    for c in cs:
        q, sc, paged, bt, cl = bench.build_workload(torch, b, h, h, 128, [c] * b, list(range(h)), dev)
        qs = torch.arange(b + 1, dtype=torch.int32, device=dev)
        out = torch.empty((b, h, 128), dtype=torch.bfloat16, device=dev)
        lse = torch.empty((b, h), dtype=torch.float32, device=dev)
        fn = lambda: kernels.context_attention(  # noqa: E731
            q, qs, paged.k_pool[0], paged.v_pool[0], cl, max_rows=1, hkv=h, block_table=bt,
            block_size=16, strides=paged.strides(), out=out, lse_out=lse)
        byt = 2 * 2 * h * 128 * b * c
        t = timed(fn, flush)
        buf = torch.empty(byt // 2, dtype=torch.bfloat16, device=dev)
        ts = timed(lambda: buf.sum(dtype=torch.float32), flush)
        print(f"c={c:5d} {byt / 1e6:7.1f} MB  ctx {t:7.1f} us {byt / t / 1e3:6.0f} GB/s   "
              f"torch.sum {ts:7.1f} us {byt / ts / 1e3:6.0f} GB/s")
        del q, sc, paged, buf


if __name__ == "__main__":
    main()
