"""Standalone system_attention (the reference `_system_attention` entry point)
at the C2-C5 system shapes: eager call time (host work included) and a CUDA
graph replay of the same call (device time: system kernel + part merge),
CUDA events, median of 10.

    python profiles/time_system_attention.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import kernels  # noqa: E402


def timed(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    for b, hq, hkv, s in ((32, 52, 52, 8192), (64, 32, 32, 4096), (128, 32, 8, 32768), (256, 64, 8, 65536)):
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(b, hq, 128, device="cuda", generator=g).to(torch.bfloat16)
        k = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
        o = torch.empty(b, hq, 128, device="cuda")
        lse = torch.empty(b, hq, device="cuda")
        call = lambda: kernels.system_attention(q, k, v, kv_layout="hsd", o_sys=o, lse_sys=lse)  # noqa: E731
        eager = timed(call)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            call()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                call()
        torch.cuda.current_stream().wait_stream(st)
        dev = timed(gr.replay)
        print(f"b={b} hq={hq} hkv={hkv} s={s}: eager {eager:7.1f} us, graph replay {dev:7.1f} us")


if __name__ == "__main__":
    main()
