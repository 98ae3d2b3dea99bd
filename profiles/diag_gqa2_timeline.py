"""Per-tile event timeline of CTA 0 of the 256-row GQA system kernel
(sys_gqa2_sm100.cu, diagnostics build: clock64 stamps).

    python profiles/diag_gqa2_timeline.py [b hq hkv s]
"""
import os
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402

NAMES = ["wg0 S ready", "wg0 P done", "wg1 S ready", "wg1 P done", "mma P0 seen", "mma S0 issued",
         "mma P1 seen", "mma S1 issued", "mma K ready", "mma V ready"]


def main():
    b, hq, hkv, s = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (128, 32, 8, 32768)))
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(b, hq, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    ts = torch.zeros(8192 * 8, dtype=torch.int64, device="cuda")
    lib = _lib.load_diag() if not os.environ.get("RB_LIB") else _lib._bind(os.environ["RB_LIB"])
    lib.rb_debug_set_timestamps.argtypes = [__import__("ctypes").c_void_p]
    if os.environ.get("RB_LIB"):
        _lib._lib = lib  # the variant library runs the kernels too
    for it in range(3):
        lib.rb_debug_set_timestamps(ts.data_ptr() if it == 2 else None)
        kernels.system_attention(q, k, v, kv_layout="hsd")
        torch.cuda.synchronize()
    lib.rb_debug_set_timestamps(None)
    t = ts[6144 * 8:6144 * 8 + 18 * 128].view(18, 128).cpu()
    t0 = int(t[t != 0].min())
    print("tile " + " ".join(f"{n:>13s}" for n in NAMES))
    for j in range(0, int(os.environ.get("ROWS", "14"))):
        print(f"{j:4d} " + " ".join(f"{(int(t[e, j]) - t0) if t[e, j] else -1:13d}" for e in range(10)))
    import statistics
    d = [int(t[1, j + 1]) - int(t[1, j]) for j in range(8, 100) if t[1, j + 1] and t[1, j]]
    if d:
        print(f"wg0 period (cycles) median {statistics.median(d)}")
    for a, bb, n in ((0, 1, "wg0 softmax"), (2, 3, "wg1 softmax")):
        x = [int(t[bb, j]) - int(t[a, j]) for j in range(8, 100) if t[a, j] and t[bb, j]]
        if x:
            print(f"{n} (S ready -> P done) median {statistics.median(x)}")
    x = [int(t[0, j + 1]) - int(t[1, j]) for j in range(8, 100) if t[0, j + 1] and t[1, j]]
    if x:
        print(f"wg0 P done -> next S ready median {statistics.median(x)}")
    # softmax phases of warp 0 of each warpgroup (diagnostics events 10-17)
    for sub in range(2):
        marks = [2 * sub, 10 + 4 * sub, 11 + 4 * sub, 12 + 4 * sub, 13 + 4 * sub, 2 * sub + 1]
        names = ["S.ld", "max", "exp+st", "wait.st", "arrive"]
        parts = []
        for a, bb, n in zip(marks, marks[1:], names):
            x = [int(t[bb, j]) - int(t[a, j]) for j in range(8, 100) if t[a, j] and t[bb, j]]
            if x:
                parts.append(f"{n} {statistics.median(x):.0f}")
        print(f"wg{sub} softmax phases (cycles): " + ", ".join(parts))
    x = [int(t[6, j]) - int(t[3, j]) for j in range(8, 100) if t[6, j] and t[3, j]]
    if x:
        print(f"wg1 warp0 P done -> MMA sees P1 median {statistics.median(x)}")
    x = [int(t[4, j]) - int(t[1, j]) for j in range(8, 100) if t[4, j] and t[1, j]]
    if x:
        print(f"wg0 warp0 P done -> MMA sees P0 median {statistics.median(x)}")


if __name__ == "__main__":
    main()
