"""Context kernel alone at C2 while a blocker kernel holds k SMs (one CTA
each, 200 KB smem, spinning -- optionally streaming HBM like the system
kernel does): does the context kernel's per-SM rate drop because it runs on
fewer SMs (its own latency chain) or because of the concurrent HBM load?
Diagnostics.

    python profiles/diag_ctx_blocked.py [c]
"""
import ctypes
import os
import statistics
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")  # the timestamped build of the kernels
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    b, h = 32, 52
    dev = torch.device("cuda", 0)
    lib = ctypes.CDLL(os.path.join(HERE, "tools", "libblocker.so"))
    lib.blocker_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                                   ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
    lib.waiter_launch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = bench.make_flush(torch, dev)
    q, sc, paged, bt, cl = bench.build_workload(torch, b, h, h, 128, [c] * b, list(range(h)), dev)
    qs = torch.arange(b + 1, dtype=torch.int32, device=dev)
    out = torch.empty((b, h, 128), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((b, h), dtype=torch.float32, device=dev)
    byt = 2 * 2 * h * 128 * b * c
    src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    from paper_2402_14808_b200.attention import RelayDecodeStep
    step = RelayDecodeStep(sc, paged, bt, cl, h, grid=kernels.sm_count(dev))
    step.system(q)
    plain = os.environ.get("DIAG_PLAIN") == "1"

    def ctx():
        # the relay step's context phase (dynamic item claims; the system
        # units count as published) unless DIAG_PLAIN=1 (static item order)
        if plain:
            kernels.context_attention(q, qs, paged.k_pool[0], paged.v_pool[0], cl, max_rows=1,
                                      hkv=h, block_table=bt, block_size=16,
                                      strides=paged.strides(), out=out, lse_out=lse)
        else:
            step.context(q)

    stamps = torch.zeros((8192, 8), dtype=torch.int64, device=dev)
    for k, stream_mb in ((0, 0), (20, 0), (40, 0), (60, 0), (40, 40), (40, 400)):
        spans = []
        for it in range(15):
            flush()
            stamps.zero_()
            _lib.load_diag().rb_debug_set_timestamps(stamps.data_ptr())
            if k:
                counter.zero_()
                ev = torch.cuda.Event()
                ev.record(main_s)
                side.wait_event(ev)
                per = stream_mb * (1 << 20) // k // 16 * 16
                lib.blocker_launch(k, 200 * 1024, 60_000, src.data_ptr() if per else None, per,
                                   counter.data_ptr(), side.cuda_stream)
                lib.waiter_launch(counter.data_ptr(), k, main_s.cuda_stream)
            ctx()
            torch.cuda.synchronize()
            _lib.load_diag().rb_debug_set_timestamps(None)
            t = stamps[1024:2048].cpu()
            t = t[t[:, 0] != 0]
            ends = [int(r[2 + w]) for r in t for w in range(4) if r[2 + w] != 0]
            sms_used = len({int(r[1]) for r in t if any(r[2 + w] != 0 for w in range(4))})
            if it >= 3:
                spans.append((max(ends) - int(t[:, 0].min())) / 1e3)
        sp = statistics.median(spans)
        print(f"c={c} blocker {k:3d} SMs streaming {stream_mb:4d} MB: ctx entry -> last compute end "
              f"{sp:6.1f} us  {byt / sp / 1e3:6.0f} GB/s  {byt / sp / 1e3 / (148 - k):5.1f} GB/s per free SM; SMs computing {sms_used}")


if __name__ == "__main__":
    main()
