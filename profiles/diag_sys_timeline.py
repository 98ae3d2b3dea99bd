"""Per-CTA timeline of the system kernel from %globaltimer stamps
(rb_debug_set_timestamps).  Prints, per s, quantiles over CTAs of each
stamp relative to the earliest CTA entry (µs), plus the event-timed launch.

    python profiles/diag_sys_timeline.py [s ...]
"""
import os
import statistics
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")  # the timestamped build of the kernels

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402

NAMES = ["entry", "prologue", "first_S", "grp0_end", "grp1_end", "kprod_end", "vprod_end", "exit"]


def run(s, b=32, h=52):
    dev = torch.device("cuda", 0)
    q = torch.randn((b, h, 128), device=dev).to(torch.bfloat16)
    k = torch.randn((h, s, 128), device=dev).to(torch.bfloat16)
    v = torch.randn((h, s, 128), device=dev).to(torch.bfloat16)
    grid = kernels.sm_count(dev)
    pk = torch.zeros((b * 8, h, 16, 128), dtype=torch.bfloat16, device=dev)
    pv = torch.zeros_like(pk)
    pst = (pk.stride(0), pk.stride(2), pk.stride(1))
    bt = torch.arange(b * 8, dtype=torch.int32, device=dev).reshape(b, 8)
    cl = torch.full((b,), 128, dtype=torch.int32, device=dev)
    qs = torch.arange(b + 1, dtype=torch.int32, device=dev)
    ts = torch.zeros((grid, 8), dtype=torch.int64, device=dev)
    import bench
    flush_fn = bench.make_flush(torch, dev)
    for it in range(4):
        flush_fn()
        _lib.load_diag().rb_debug_set_timestamps(ts.data_ptr() if it == 3 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if MODE == "relay":  # system kernel as it runs inside rb_relay_attention
            kernels.relay_attention(q, qs, k, v, pk, pv, cl, max_rows=1, hkv=h, sys_layout="hsd",
                                    block_table=bt, block_size=16, strides=pst, grid=grid,
                                    phases=1)
        else:
            kernels.system_attention(q, k, v, kv_layout="hsd", grid=grid)
        e1.record()
        torch.cuda.synchronize()
    _lib.load_diag().rb_debug_set_timestamps(None)
    t = ts.cpu().double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"s={s}: event {e0.elapsed_time(e1) * 1e3:.1f} us; plan {_lib.sys_plan(b, h, h, s, grid)[0]}")
    for i, n in enumerate(NAMES):
        col = sorted(rel[:, i].tolist())
        print(f"  {n:10s} min {col[0]:7.1f} p50 {col[len(col)//2]:7.1f} p90 {col[int(len(col)*.9)]:7.1f} max {col[-1]:7.1f}")
    dur = (t[:, 7] - t[:, 0]) / 1e3
    print(f"  cta duration p50 {statistics.median(dur.tolist()):.1f} max {dur.max().item():.1f}")


MODE = os.environ.get("DIAG_MODE", "relay")

if __name__ == "__main__":
    for s in [int(x) for x in (sys.argv[1:] or ["512", "8192"])]:
        run(s)
