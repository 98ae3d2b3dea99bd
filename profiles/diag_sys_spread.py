import os, sys, torch
os.environ.setdefault("RB_DIAG", "1")
sys.path.insert(0, "/root/repo")
import bench
from paper_2402_14808_b200 import _lib, kernels
from paper_2402_14808_b200.attention import RelayDecodeStep
dev = torch.device("cuda", 0)
s = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
q, sc, paged, bt, cl = bench.build_workload(torch, 32, 52, 52, s, [128] * 32, list(range(52)), dev)
flush = bench.make_flush(torch, dev)
step = RelayDecodeStep(sc, paged, bt, cl, 52)
ts = torch.zeros((8192, 8), dtype=torch.int64, device=dev)
res = []
for it in range(6):
    flush(); ts.zero_()
    _lib.load_diag().rb_debug_set_timestamps(ts.data_ptr() if it >= 3 else None)
    step(q); torch.cuda.synchronize()
    if it >= 3:
        t = ts.cpu()
        sys_t = t[:1024][t[:1024, 0] != 0]
        t0 = int(sys_t[:, 0].min())
        rows = [(int(r[1]), (int(r[7]) - t0) / 1e3, int(r[4]), (int(r[2]) - t0) / 1e3) for r in sys_t]
        res.append(rows)
_lib.load_diag().rb_debug_set_timestamps(None)
P = step.plan
print("plan", P)
for rows in res:
    ex = sorted(r[1] for r in rows)
    print("exit p0 %.1f p50 %.1f p90 %.1f max %.1f" % (ex[0], ex[len(ex)//2], ex[int(len(ex)*.9)], ex[-1]))
# per CTA index (order of sys_t rows = blockIdx) exits across the 3 runs
import statistics
n = len(res[0])
avg = [statistics.mean(res[k][i][1] for k in range(3)) for i in range(n)]
order = sorted(range(n), key=lambda i: -avg[i])
print("slowest CTAs (idx: mean exit, units, sm):", [(i, round(avg[i],1), res[0][i][2], res[0][i][0]) for i in order[:10]])
print("fastest:", [(i, round(avg[i],1), res[0][i][2], res[0][i][0]) for i in order[-5:]])
by_units = {}
for i in range(n):
    by_units.setdefault(res[0][i][2], []).append(avg[i])
print({u: (len(v), round(statistics.mean(v),1)) for u, v in by_units.items()})
# consistency: correlation of exit between runs
import itertools
for a, b in [(0,1),(1,2)]:
    xa = [res[a][i][1] for i in range(n)]; xb = [res[b][i][1] for i in range(n)]
    ma, mb = statistics.mean(xa), statistics.mean(xb)
    cov = sum((x-ma)*(y-mb) for x,y in zip(xa,xb)); va = sum((x-ma)**2 for x in xa); vb = sum((y-mb)**2 for y in xb)
    print("run corr", a, b, round(cov/(va*vb)**.5, 2))
