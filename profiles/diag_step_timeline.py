"""Per-CTA timeline of the one-kernel relay step (rb_relay_step) from
%globaltimer stamps (rb_debug_set_timestamps, [grid][64] u64 per launch).

    python profiles/diag_step_timeline.py s phases [cta ...]

Prints quantiles over CTAs of entry / prologue / first S / softmax end /
epilogue end / exit, and for the listed CTAs the softmax S-arrival time of
each tile and the epilogue start/end of each part (us from the first entry).
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
phases = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctas = [int(x) for x in sys.argv[3:]] or [0, 60, 147]
dev = torch.device("cuda", 0)
q, relay, naive, paged, bt = bench.build(torch, s, list(range(bench.H)), dev)
flush = bench.make_flush(torch, dev)
grid = relay.grid
ts = torch.zeros((grid, 512), dtype=torch.int64, device=dev)
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
print(f"s={s} phases={phases}: event {e0.elapsed_time(e1) * 1e3:.1f} us")
for i, n in enumerate(["entry", "prologue", "first_S", "softmax_end", "epi_end", "exit"]):
    col = sorted(rel[:, i].tolist())
    print(f"  {n:12s} min {col[0]:7.1f} p50 {col[len(col)//2]:7.1f} p90 {col[int(len(col)*.9)]:7.1f} max {col[-1]:7.1f}")
def row(c, a, n=32):
    return " ".join(f"{x:.1f}" for x in rel[c, a:a + n].tolist() if x > 0)


for c in ctas:
    if c >= grid:
        continue
    print(f"  cta {c}:")
    print(f"    K prod loop top      {row(c, 360)}")
    print(f"    K prod after ids     {row(c, 392)}")
    print(f"    K prod after stage   {row(c, 424)}")
    print(f"    K prod after Q       {row(c, 456)}")
    print(f"    K prod before-wait   {row(c, 168)}")
    print(f"    K prod after-wait    {row(c, 136)}")
    print(f"    V prod after-wait    {row(c, 232)}")
    print(f"    QK issue             {row(c, 264)}")
    print(f"    softmax S arrival    {row(c, 8)}")
    print(f"    softmax P ready      {row(c, 328)}")
    print(f"    PV issue             {row(c, 296)}")
    print(f"    epilogue part start  {row(c, 40)}")
    print(f"    epilogue after ld    {row(c, 72)}")
    print(f"    epilogue after hand  {row(c, 200)}")
    print(f"    epilogue part end    {row(c, 104)}")
