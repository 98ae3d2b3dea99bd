"""Per-SM timeline of one relay decode step (system kernel + paged context
kernel with the fused epilogue) from %globaltimer stamps
(rb_debug_set_timestamps).  Diagnostics only.

    python profiles/diag_relay_timeline.py [s] [phases]

System CTA stamps [1024][8]: entry, smid, first_S, grp0_end, grp1_end,
kprod_end, vprod_end, exit.  Extended system startup stamps at offset 2048*8: prologue, first K
issue, Q ready, first K full, first MMA, first V issue.  Context CTA stamps
start at offset 1024*8:
entry, smid, warp0..3 compute end, after-PDL-wait, exit.
"""
import os
import statistics
import sys

import torch

os.environ.setdefault("RB_DIAG", "1")  # the timestamped build of the kernels

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import _lib, kernels  # noqa: E402


def q(col):
    col = sorted(col)
    n = len(col)
    return f"min {col[0]:6.1f} p10 {col[n // 10]:6.1f} p50 {col[n // 2]:6.1f} p90 {col[int(n * .9)]:6.1f} max {col[-1]:6.1f}"


def run(s, phases=3, b=32, h=52, c=128, hkv=None):
    hkv = h if hkv is None else hkv
    dev = torch.device("cuda", 0)
    qq = torch.randn((b, h, 128), device=dev).to(torch.bfloat16)
    k = torch.randn((hkv, s, 128), device=dev).to(torch.bfloat16)
    v = torch.randn((hkv, s, 128), device=dev).to(torch.bfloat16)
    nblk = c // 16
    grid = int(os.environ.get("DIAG_GRID", "0")) or _lib.relay_sys_grid(b, h, hkv, s, b * c, kernels.sm_count(dev))
    pk = torch.randn((b * nblk, hkv, 16, 128), device=dev).to(torch.bfloat16)
    pv = torch.randn_like(pk)
    pst = (pk.stride(0), pk.stride(2), pk.stride(1))
    bt = torch.randperm(b * nblk, device=dev).to(torch.int32).reshape(b, nblk)
    if os.environ.get("DIAG_SEQBT"):
        bt = torch.arange(b * nblk, device=dev, dtype=torch.int32).reshape(b, nblk)
    cl = torch.full((b,), c, dtype=torch.int32, device=dev)
    if os.environ.get("DIAG_CLENS_U"):
        # C3-style context lengths ~ U[lo, hi] (seeded), in a c-token block table
        lo, hi = (int(x) for x in os.environ["DIAG_CLENS_U"].split(","))
        import numpy as np
        lens = np.random.default_rng(1002).integers(lo, hi + 1, size=b)
        cl = torch.tensor(lens, dtype=torch.int32, device=dev)
    qs = torch.arange(b + 1, dtype=torch.int32, device=dev)
    # DIAG_ORDER=1: claim the context work longest request first (RelayDecodeStep's req_order)
    order = (torch.argsort(cl, descending=True, stable=True).to(torch.int32)
             if os.environ.get("DIAG_ORDER") else None)
    ts = torch.zeros((8192, 8), dtype=torch.int64, device=dev)
    import bench
    flush_fn = bench.make_flush(torch, dev)
    for it in range(5):
        if not os.environ.get("DIAG_NOFLUSH"):
            flush_fn()
        ts.zero_()
        _lib.load_diag().rb_debug_set_timestamps(ts.data_ptr() if it == 4 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kernels.relay_attention(qq, qs, k, v, pk, pv, cl, max_rows=h // hkv, hkv=hkv, sys_layout="hsd",
                                block_table=bt, block_size=16, strides=pst, grid=grid,
                                phases=phases, req_order=order,
                                max_ctx_len=c if os.environ.get("DIAG_SPLIT") else 0)
        e1.record()
        torch.cuda.synchronize()
    _lib.load_diag().rb_debug_set_timestamps(None)
    t = ts.cpu()
    sys_t = t[:1024][t[:1024, 0] != 0]
    ctx_t = t[1024:2048][t[1024:2048, 0] != 0]
    starts = []
    if len(sys_t):
        starts.append(int(sys_t[:, 0].min()))
    if len(ctx_t):
        starts.append(int(ctx_t[:, 0].min()))
    t0 = min(starts)
    us = lambda x: (int(x) - t0) / 1e3  # noqa: E731
    print(f"s={s} phases={phases} sys grid {grid}: event {e0.elapsed_time(e1) * 1e3:.1f} us")
    sys_exit = {}
    if len(sys_t):
        for i, n in [(0, "entry"), (2, "first_S"), (3, "softmax_end"), (5, "kprod_end"), (6, "vprod_end"), (7, "exit")]:
            col = [us(r[i]) for r in sys_t]
            print(f"  sys {n:10s} {q(col)}")
        ext = t[2048:3072][t[2048:3072, 0] != 0]
        for i, n in enumerate(["prologue", "k0_issue", "q_ready", "k0_full", "mma0", "v0_issue"]):
            col = [us(r[i]) for r in ext if r[i] != 0]
            if col:
                print(f"  sys {n:10s} {q(col)}")
        if len(ext):
            print(f"  sys units/CTA       {q([float(v) for v in sys_t[:, 4].tolist()])}")
            for c, n in ((6, "epi o_full wait"), (7, "epi thru row sums"), (3, "epi total")):
                print(f"  sys {n:17s} {q([float(v) / 1e3 for v in ext[:, c].tolist()])}")
        for r in sys_t:
            sys_exit[int(r[1])] = us(r[7])
    if len(ctx_t):
        print(f"  ctx CTAs {len(ctx_t)}")
        print(f"  ctx entry      {q([us(r[0]) for r in ctx_t])}")
        ce = [us(r[2 + w]) for r in ctx_t for w in range(4) if r[2 + w] != 0]
        print(f"  ctx warp compute end {q(ce)}")
        pw = [us(r[6]) for r in ctx_t if r[6] != 0]
        if pw:
            print(f"  ctx after pdl wait   {q(pw)}")
        print(f"  ctx exit       {q([us(r[7]) for r in ctx_t])}")
        per_sm = {}
        for r in ctx_t:
            per_sm.setdefault(int(r[1]), []).append(r)
        cnt = [len(v_) for v_ in per_sm.values()]
        print(f"  ctx CTAs per SM: {sorted(set(cnt))} (SMs used {len(per_sm)}), hist "
              + str({k_: cnt.count(k_) for k_ in sorted(set(cnt))}))
        last = sorted(per_sm.items(), key=lambda kv: max(us(r[7]) for r in kv[1]))
        for sm, rows in last[-6:] + last[:3]:
            print(f"    sm {sm:3d}: sys exit {sys_exit.get(sm, float('nan')):6.1f}; ctx entries "
                  + ", ".join(f"{us(r[0]):.1f}" for r in rows) + "; compute ends "
                  + ", ".join(f"{us(r[2 + w]):.1f}" for r in rows for w in range(4) if r[2 + w])
                  + "; exits " + ", ".join(f"{us(r[7]):.1f}" for r in rows))
        acc = t[4096:4096 + 1024][t[4096:4096 + 1024, 1] != 0]
        if len(acc):
            names = ["merger m_full wait", "merger items", "merger work", "w0 i_full wait",
                     "w0 m_empty wait", "merger i_meta wait"]
            print(f"  ctx end-phase start  {q([us(v) for v in acc[:, 6].tolist()])}")
            print(f"  ctx deferred rows    {q([float(v) for v in acc[:, 7].tolist()])}")
            for i, n in enumerate(names):
                col = [float(v) / (1 if i == 1 else 1e3) for v in acc[:, i].tolist()]
                print(f"  ctx {n:20s} {q(col)}")
        wst = t[6144:6144 + 1024][t[6144:6144 + 1024, 4] != 0]
        if len(wst):
            for i, n in enumerate(["w0 in try_issue", "w0 data wait", "w0 compute"]):
                print(f"  ctx {n:20s} {q([float(v) / 1e3 for v in wst[:, i].tolist()])}")
            print(f"  ctx w0 chunks        {q([float(v) for v in wst[:, 4].tolist()])}")
            print(f"  ctx w0 waits w/ 1 in flight {q([float(v) for v in wst[:, 3].tolist()])}")
        # early (started beside the system kernel) vs late context CTAs
        accf = t[4096:4096 + 1024]
        ctx_idx = [i for i in range(1024) if int(t[1024 + i, 0]) != 0]
        if len(ctx_idx) and int(accf[:, 6].max()) != 0:
            early = [i for i in ctx_idx if us(t[1024 + i, 0]) < 50.0]
            late = [i for i in ctx_idx if us(t[1024 + i, 0]) >= 50.0]
            for name, grp in (("early", early), ("late", late)):
                if not grp:
                    continue
                ep = [us(accf[i, 6]) for i in grp if int(accf[i, 6])]
                dn = [us(t[1024 + i, 6]) for i in grp if int(t[1024 + i, 6])]
                nd = [float(accf[i, 7]) for i in grp]
                print(f"  ctx {name} CTAs {len(grp)}: end-phase start {q(ep) if ep else '-'}")
                print(f"  ctx {name} done {q(dn) if dn else '-'}; deferred {q(nd)}")
        durs = [(int(r[7]) - int(r[0])) / 1e3 for r in ctx_t]
        print(f"  ctx CTA duration p50 {statistics.median(durs):.1f} max {max(durs):.1f}")


if __name__ == "__main__":
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    ph = [int(sys.argv[2])] if len(sys.argv) > 2 else [3, 2]
    # optional workload: b h hkv c (default C2: 32 52 52 128)
    b, h, hkv, c = (int(x) for x in sys.argv[3:7]) if len(sys.argv) > 6 else (32, 52, 52, 128)
    for p in ph:
        run(s, p, b=b, h=h, c=c, hkv=hkv)
