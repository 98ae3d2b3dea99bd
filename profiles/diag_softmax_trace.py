"""Per-tile trace of the relay step's MMA issuers and softmax groups for one
CTA (build with -DRB_STEP_TRACE=1):
    python profiles/diag_softmax_trace.py s phases cta
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib  # noqa: E402

s, phases, cta = (int(x) for x in sys.argv[1:4])
dev = torch.device("cuda", 0)
q, relay, naive, paged, bt = bench.build(torch, s, list(range(bench.H)), dev)
flush = bench.make_flush(torch, dev)
ts = torch.zeros((relay.grid, 512), dtype=torch.int64, device=dev)
for it in range(4):
    flush()
    _lib.load().rb_debug_set_timestamps(ts.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    relay._launch(q, phases)
    e1.record()
    torch.cuda.synchronize()
_lib.load().rb_debug_set_timestamps(None)
t = ts.cpu().double()
t0 = t[:, 0].min()
rel = torch.where(t > 0, (t - t0) / 1e3, torch.zeros_like(t))
print(f"event {e0.elapsed_time(e1) * 1e3:.1f} us")
for i, nm in enumerate(["entry", "prologue", "first S", "grp0 end", "grp1 end", "exit-ish", "barrier", "exit"]):
    col = sorted(rel[:, i].tolist())
    print(f"  {nm:10s} p10 {col[len(col) // 10]:6.1f} p50 {col[len(col) // 2]:6.1f} max {col[-1]:6.1f}")
for nm, base in [("QK issue", 264), ("S arrival", 8), ("pass1 done", 360), ("red_or", 392),
                 ("rare done", 424), ("p_empty ok", 456), ("P arrived", 40), ("pe reduced", 136),
                 ("pe bar", 168), ("pe o_full", 200), ("tile done", 328), ("PV issue", 296)]:
    print(f"{nm:11s}", " ".join(f"{x:5.1f}" for x in rel[cta, base:base + 24].tolist()))
# per-CTA imbalance: group end time vs SM id
ends = torch.maximum(rel[:, 3], rel[:, 4])
smid = t[:, 480].long()
order = torch.argsort(ends)
print("fastest CTAs (cta:sm:end):", [(int(c), int(smid[c]), round(float(ends[c]), 1)) for c in order[:12]])
print("slowest CTAs (cta:sm:end):", [(int(c), int(smid[c]), round(float(ends[c]), 1)) for c in order[-12:]])
lo = ends[smid < 74].mean().item(); hi = ends[smid >= 74].mean().item()
ev = ends[smid % 2 == 0].mean().item(); od = ends[smid % 2 == 1].mean().item()
print(f"mean end: sm<74 {lo:.1f} sm>=74 {hi:.1f}; even sm {ev:.1f} odd sm {od:.1f}")
print("work tiles per CTA (sys) const; end-time by cta index quartile:",
      [round(ends[i * len(ends) // 4:(i + 1) * len(ends) // 4].mean().item(), 1) for i in range(4)])
