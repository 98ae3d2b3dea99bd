"""Compare the event-timed duration of a graph-replayed relay step with the
span of its kernels (first CTA entry to last CTA exit, %globaltimer stamps),
to see how much of the step is launch / completion overhead.  Diagnostics.

    python profiles/diag_graph_overhead.py [s ...]
"""
import os
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")  # the timestamped build of the kernels

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    flush = bench.make_flush(torch, dev)
    for s in [int(x) for x in (sys.argv[1:] or ["512", "8192"])]:
        q, relay, _, _, _ = bench.build(torch, s, list(range(bench.H)), dev)
        ts = torch.zeros((3072, 8), dtype=torch.int64, device=dev)
        _lib.load_diag().rb_debug_set_timestamps(ts.data_ptr())
        phases = int(os.environ.get("DIAG_PHASES", "3"))
        fn = {3: lambda: relay(q), 1: lambda: relay.system(q), 2: lambda: relay.context(q)}[phases]
        g = bench.graph_of(torch, fn)
        rows = []
        for _ in range(10):
            if not os.environ.get("DIAG_NOFLUSH"):
                flush()
            ts.zero_()
            # a marker kernel right before the graph: its end is the start
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            t = ts.cpu()
            sysr = t[:1024][t[:1024, 0] != 0]
            ctx = t[1024:2048][t[1024:2048, 0] != 0]
            firsts = [int(x[:, 0].min()) for x in (sysr, ctx) if len(x)]
            lasts = [int(sysr[:, 7].max())] if len(sysr) else []
            if len(ctx):
                lasts += [int(ctx[:, 7].max()), int(ctx[:, 6].max())]
            first, last = min(firsts), max(lasts)
            rows.append((e0.elapsed_time(e1) * 1e3, (last - first) / 1e3))
        _lib.load_diag().rb_debug_set_timestamps(None)
        rows.sort()
        ev, span = rows[len(rows) // 2]
        # reference: a graph of one trivial kernel
        x = torch.zeros(1024, device=dev)
        gt = bench.graph_of(torch, lambda: x.add_(1.0))
        triv = []
        for _ in range(10):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gt.replay()
            e1.record()
            torch.cuda.synchronize()
            triv.append(e0.elapsed_time(e1) * 1e3)
        print(f"  trivial-kernel graph: {sorted(triv)[5]:.1f} us")
        print(f"s={s} phases={phases}: graph step event {ev:.1f} us, kernel span {span:.1f} us, "
              f"outside kernels {ev - span:.1f} us", flush=True)


if __name__ == "__main__":
    main()
