"""Break the e2e decode step (bench.py e2e, C2 s=8192) into its parts:
CUDA-graph replays after the bench's L2 flush, CUDA events.  Diagnostics.

    python profiles/diag_e2e.py [s]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    B, H, C, D = bench.B, bench.H, bench.C, bench.D
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    q, sc, paged, bt, cl = bench.build_workload(torch, B, H, H, s, [C] * B, list(range(H)), dev)
    step = RelayDecodeStep(sc, paged, bt, cl, H)
    qkv_h = torch.randn((3, B, H, D)).to(torch.bfloat16).pin_memory()
    out_h = torch.empty((B, H, D), dtype=torch.bfloat16).pin_memory()
    qkv_d = torch.empty_like(qkv_h, device=dev)
    btc = bt.cpu()
    slots = torch.tensor([int(btc[r, (C - 1) // 16]) * 16 + (C - 1) % 16 for r in range(B)],
                         dtype=torch.int32, device=dev)

    def timed(fn):
        g = bench.graph_of(torch, fn)
        return statistics.median(bench.time_loop(torch, g.replay, 30, 3, flush)) * 1e3

    parts = {
        "H2D q|k|v (1.28 MB)": lambda: qkv_d.copy_(qkv_h, non_blocking=True),
        "H2D q (0.43 MB)": lambda: qkv_d[0].copy_(qkv_h[0], non_blocking=True),
        "D2H out (0.43 MB)": lambda: out_h.copy_(step.out, non_blocking=True),
        "append": lambda: paged.append_slots(0, qkv_d[1], qkv_d[2], slots),
        "relay step": lambda: step(qkv_d[0]),
    }
    for name, fn in parts.items():
        print(f"{name:22s} {timed(fn):7.1f} us")
    qh, kh, vh = qkv_h[0], qkv_h[1], qkv_h[2]
    kd, vd = qkv_d[1], qkv_d[2]
    zc = {
        "step, q from host": lambda: step._launch(qh, 3),
        "step, out to host": lambda: step._launch(qkv_d[0], 3, out=out_h),
        "step + fused append (device k/v)": lambda: step._launch(qkv_d[0], 3, k_new=kd, v_new=vd,
                                                                 slot_mapping=slots),
        "step + fused append (host k/v)": lambda: step._launch(qkv_d[0], 3, k_new=kh, v_new=vh,
                                                               slot_mapping=slots),
    }
    for name, fn in zc.items():
        print(f"{name:34s} {timed(fn):7.1f} us")
    for zcopy in (False, True):
        replay = step.host_step_graph(qkv_h, slots, out_h, zero_copy=zcopy)
        ts = sorted(x * 1e3 for x in bench.time_loop(torch, replay, 50, 5, flush))
        print(f"e2e graph zero_copy={zcopy}: median {ts[25]:7.1f} mean {statistics.mean(ts):7.1f} "
              f"min {ts[0]:7.1f} max {ts[-1]:7.1f} us")
    return
    replay = step.host_step_graph(qkv_h, slots, out_h)
    print(f"{'e2e graph':22s} {statistics.median(bench.time_loop(torch, replay, 30, 3, flush)) * 1e3:7.1f} us")


if __name__ == "__main__":
    main()
