"""Per-role event trace of system-kernel CTA 0 (diagnostics build, clock64):
K / V producers (slot free), Q.K^T issuer (K landed, S buffer free), P.V
issuer (V landed, P ready), softmax warps (S ready, max flags exchanged,
exponentials done, P buffer free, P published).

    python profiles/diag_sys_trace.py [s] [grid]
"""
import os
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402

NAMES = {10: "Kslot", 20: "Vslot", 30: "Kfull", 31: "Sfree", 40: "Vfull", 41: "Pfull",
         50: "S", 51: "flag", 52: "exp", 53: "Pfree", 54: "Ppub"}
GHZ = 1.965


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    b, h, c = 32, 52, 128
    dev = torch.device("cuda", 0)
    q, sc, paged, bt, cl = bench.build_workload(torch, b, h, h, s, [c] * b, list(range(h)), dev)
    flush = bench.make_flush(torch, dev)
    step = RelayDecodeStep(sc, paged, bt, cl, h, grid=grid or None)
    ts = torch.zeros((8192, 8), dtype=torch.int64, device=dev)
    for it in range(4):
        flush()
        ts.zero_()
        _lib.load_diag().rb_debug_set_timestamps(ts.data_ptr() if it == 3 else None)
        step(q)
        torch.cuda.synchronize()
    _lib.load_diag().rb_debug_set_timestamps(None)
    t = ts.cpu().reshape(-1)
    base = 3072 * 8
    evs = []
    for w in range(12):
        for n in range(256):
            clk, code = int(t[base + w * 512 + 2 * n]), int(t[base + w * 512 + 2 * n + 1])
            if clk == 0:
                break
            evs.append((clk, w, code))
    t0 = min(e[0] for e in evs)
    print(f"s={s} grid={step.grid} plan={step.plan}")
    for w in range(12):
        line = [f"{(clk - t0) / GHZ / 1e3:5.2f}:{NAMES.get(code // 10000, '?')}{code % 10000}"
                for clk, ww, code in evs if ww == w]
        if not line:
            continue
        print(f"--- warp {w} ({len(line)} events)")
        for i in range(0, min(len(line), 64), 8):
            print("   " + "  ".join(line[i:i + 8]))


if __name__ == "__main__":
    main()
