"""Context split-K on few long contexts (b = 2, 8 KV heads, 32 query heads,
c = 32768): context attention with and without the split (max_ctx_len given
or 0), CUDA-graph replay after the bench's L2 flush.  Diagnostics.

    python profiles/diag_ctx_split.py [b c]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import kernels  # noqa: E402


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    c = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    hq, hkv = 32, 8
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    q, sc, paged, bt, cl = bench.build_workload(torch, b, hq, hkv, 128, [c] * b, list(range(hkv)), dev)
    qs = torch.arange(b + 1, dtype=torch.int32, device=dev)
    byt = 2 * 2 * hkv * 128 * b * c
    for name, mcl in (("split-K", bt.shape[1] * paged.block_size), ("no split", 0)):
        fn = lambda: kernels.context_attention(  # noqa: E731
            q, qs, paged.k_pool[0], paged.v_pool[0], cl, max_rows=hq // hkv, hkv=hkv,
            block_table=bt, block_size=16, strides=paged.strides(), max_ctx_len=mcl)
        fn()
        g = bench.graph_of(torch, fn)
        t = statistics.median(bench.time_loop(torch, g.replay, 20, 3, flush)) * 1e3
        print(f"b={b} c={c} {name:8s}: {t:7.1f} us  {byt / t / 1e3:6.0f} GB/s of {byt / 1e6:.0f} MB")


if __name__ == "__main__":
    main()
