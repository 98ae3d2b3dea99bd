"""Per-CTA phases of the 256-row GQA system kernel run alone (diagnostics
build, %globaltimer): entry, first S, last unit's epilogue start, part
written, merge done, exit -- where a C4/C5 launch spends its time beyond the
key-tile loop.

    python profiles/diag_gqa2_spread.py [b hq hkv s [grid]]
"""
import os
import statistics
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    b, hq, hkv, s = a[:4] if len(a) >= 4 else (128, 32, 8, 32768)
    grid = a[4] if len(a) > 4 else None
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(b, hq, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    ts = torch.zeros(8192 * 8, dtype=torch.int64, device="cuda")
    lib = _lib.load_diag() if not os.environ.get("RB_LIB") else _lib._bind(os.environ["RB_LIB"])
    lib.rb_debug_set_timestamps.argtypes = [__import__("ctypes").c_void_p]
    _lib._lib = lib
    print("plan", _lib.sys_plan(b, hq, hkv, s, grid or kernels.sm_count(q.device))[0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(4):
        ts.zero_()
        lib.rb_debug_set_timestamps(ts.data_ptr() if it == 3 else None)
        e0.record()
        kernels.system_attention(q, k, v, kv_layout="hsd", grid=grid)
        e1.record()
        torch.cuda.synchronize()
    lib.rb_debug_set_timestamps(None)
    print(f"kernel {e0.elapsed_time(e1) * 1e3:.1f} us (events, diagnostics build)")
    t = ts.view(8192, 8)[:1024].cpu()
    rows = t[t[:, 0] != 0]
    t0 = int(rows[:, 0].min())
    us = lambda c: [(int(r[c]) - t0) / 1e3 for r in rows if int(r[c]) != 0]  # noqa: E731
    for name, c in (("entry", 0), ("Q loaded", 6), ("first S", 2), ("epilogue", 3), ("part written", 4), ("merged", 5),
                    ("exit", 7)):
        x = sorted(us(c))
        if x:
            print(f"{name:13s} n={len(x):4d} min {x[0]:7.1f} p50 {statistics.median(x):7.1f} "
                  f"max {x[-1]:7.1f} us")
    d = [(int(r[5]) - int(r[4])) / 1e3 for r in rows if int(r[5]) and int(r[4])]
    if d:
        print(f"merge duration p50 {statistics.median(d):.1f} max {max(d):.1f} us")
    d = sorted((int(r[3]) - int(r[2])) / 1e3 for r in rows if int(r[3]) and int(r[2]))
    if d:
        print(f"first S -> last epilogue p10 {d[len(d) // 10]:.1f} p50 {statistics.median(d):.1f} "
              f"max {d[-1]:.1f} us (key-tile loop of the CTA's range)")
    d = [(int(r[4]) - int(r[3])) / 1e3 for r in rows if int(r[4]) and int(r[3])]
    if d:
        print(f"part write p50 {statistics.median(d):.1f} max {max(d):.1f} us")


if __name__ == "__main__":
    main()
