"""Per-warp event trace of context CTAs 0 and 1 (diagnostics build, clock64):
scheduler claims / publications, worker issue / data-ready / compute / item
start / handoff, merger waits.  Prints each warp's events with the time since
the CTA's first event.

    python profiles/diag_ctx_trace.py [s] [phases] [cta] [b hq hkv c]
"""
import os
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402
from paper_2402_14808_b200.attention import RelayDecodeStep  # noqa: E402

NAMES = {10: "iss>", 11: "iss<", 21: "data", 30: "comp", 40: "item", 50: "hand",
         60: "S.claim", 61: "S.slot", 62: "S.got", 70: "M.wait", 71: "M.full", 72: "M.done"}
GHZ = 1.965


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    phases = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cta = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    b, h, hkv, c = (int(x) for x in sys.argv[4:8]) if len(sys.argv) > 7 else (32, 52, 52, 128)
    dev = torch.device("cuda", 0)
    q, sc, paged, bt, cl = bench.build_workload(torch, b, h, hkv, s, [c] * b, list(range(hkv)), dev)
    flush = bench.make_flush(torch, dev)
    step = RelayDecodeStep(sc, paged, bt, cl, h)
    ts = torch.zeros((8192, 8), dtype=torch.int64, device=dev)
    # RB_LIB: a diagnostics variant (built with -DRB_DIAG=1) runs the kernels
    # and takes the timestamp buffer itself
    diag = _lib.load_diag() if not os.environ.get("RB_LIB") else _lib.load()
    diag.rb_debug_set_timestamps.argtypes = [__import__("ctypes").c_void_p]
    for it in range(4):
        if phases == 2:
            step.system(q)
        flush()
        ts.zero_()
        diag.rb_debug_set_timestamps(ts.data_ptr() if it == 3 else None)
        step._launch(q, phases)
        torch.cuda.synchronize()
    diag.rb_debug_set_timestamps(None)
    t = ts.cpu().reshape(-1)
    base = 7168 * 8 + cta * 6 * 512
    evs = []
    for w in range(6):
        for n in range(256):
            clk = int(t[base + w * 512 + 2 * n])
            code = int(t[base + w * 512 + 2 * n + 1])
            if clk == 0:
                break
            evs.append((clk, w, code))
    t0 = min(e[0] for e in evs)
    for w in range(6):
        role = "sched" if w == 0 else "merger" if w == 5 else f"worker{w - 1}"
        line = []
        for clk, ww, code in evs:
            if ww != w:
                continue
            line.append(f"{(clk - t0) / GHZ / 1e3:5.2f}:{NAMES.get(code // 10000, '?')}{code % 10000}")
        print(f"--- CTA {cta} {role} ({len(line)} events)")
        for i in range(0, min(len(line), int(os.environ.get("MAXEV", "96"))), 8):
            print("   " + "  ".join(line[i:i + 8]))


if __name__ == "__main__":
    main()
