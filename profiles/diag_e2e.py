"""Break the e2e decode step (bench.py e2e) into its parts, event-timed.
    python profiles/diag_e2e.py
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def t(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def main():
    dev = torch.device("cuda", 0)
    q, relay, naive, paged, bt = bench.build(torch, 8192, list(range(bench.H)), dev)
    B, H, D = bench.B, bench.H, bench.D
    qkv_h = torch.randn((3, B, H, D)).to(torch.bfloat16).pin_memory()
    out_h = torch.empty((B, H, D), dtype=torch.bfloat16).pin_memory()
    qkv_d = torch.empty((3, B, H, D), dtype=torch.bfloat16, device=dev)
    slots = torch.arange(B, dtype=torch.int32, device=dev) * 16
    print(f"H2D {qkv_h.numel()*2} B: {t(lambda: qkv_d.copy_(qkv_h, non_blocking=True)):.1f} us")
    print(f"D2H {out_h.numel()*2} B: {t(lambda: out_h.copy_(relay.out, non_blocking=True)):.1f} us")
    print(f"append: {t(lambda: paged.append_slots(0, qkv_d[1], qkv_d[2], slots)):.1f} us")
    print(f"relay step: {t(lambda: relay(q)):.1f} us")
    print(f"system only: {t(lambda: relay.system(q)):.1f} us")
    print(f"context only: {t(lambda: relay.context(q)):.1f} us")
    print(f"step_host eager: {t(lambda: relay.step_host(qkv_h[0], qkv_h[1], qkv_h[2], slots, out_h)):.1f} us")
    g = relay.host_step_graph(qkv_h, slots, out_h)
    print(f"host_step_graph: {t(g):.1f} us")


if __name__ == "__main__":
    main()
