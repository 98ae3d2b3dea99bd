"""Per-source-line view of an ncu report: instructions executed and warp
stall samples (with the top stall reasons) of one kernel, aggregated by the
CUDA source line the SASS maps to (nvdisasm -g line info of our own .so).

    python profiles/ncu_lines.py <report.ncu-rep> <kernel-substring> [top]

Diagnostics (run in the build container; the report comes from gpurun).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2402_14808_b200", "librelay_b200.so")


def sass_lines(kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    out = []
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        text = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, f)], capture_output=True,
                              text=True).stdout.splitlines()
        starts = [i for i, l in enumerate(text) if l.startswith(".text.") and kernel_sub in l and l.endswith(":")]
        if not starts:
            continue
        cur = None
        for l in text[starts[0] + 1:]:
            if l.startswith("//---"):
                break
            m = re.search(r"line (\d+)", l)
            if "//## File" in l and m:
                cur = (l.split('"')[1].split("/")[-1], int(m.group(1)))
            if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
                out.append(cur)
        return out
    raise SystemExit(f"kernel {kernel_sub} not found in {LIB}")


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    by_inst = len(sys.argv) > 4 and sys.argv[4] == "inst"  # rank lines by instructions executed
    csv_text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                              capture_output=True, text=True).stdout
    rows = list(csv.reader(csv_text.splitlines()))
    hdr = rows[1]
    ix = hdr.index("Instructions Executed")
    iw = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    data = [r for r in rows[2:] if len(r) > ix]
    locs = sass_lines(ksub)
    if len(locs) != len(data):
        print(f"warning: {len(locs)} SASS lines vs {len(data)} profiled instructions")
    inst, samp = collections.Counter(), collections.Counter()
    stalls = collections.defaultdict(collections.Counter)
    for r, loc in zip(data, locs):
        inst[loc] += int(r[ix] or 0)
        samp[loc] += int(r[iw] or 0)
        for c in stall_cols:
            try:
                stalls[loc][hdr[c][6:]] += int(r[c] or 0)
            except ValueError:
                pass
    tot_i, tot_s = sum(inst.values()), sum(samp.values())
    srcs = {}
    print(f"instructions {tot_i}, stall samples {tot_s}")
    ranked = [(loc, samp[loc]) for loc, _ in inst.most_common(top)] if by_inst else samp.most_common(top)
    for loc, s in ranked:
        if loc is None:
            continue
        f, ln = loc
        if f not in srcs:
            path = os.path.join(ROOT, "paper_2402_14808_b200", "csrc", f)
            srcs[f] = open(path).read().splitlines() if os.path.exists(path) else []
        text = srcs[f][ln - 1].strip() if ln - 1 < len(srcs[f]) else "?"
        reasons = ", ".join(f"{k} {v}" for k, v in stalls[loc].most_common(3) if v)
        print(f"{f}:{ln:<5d} samp {s:6d} ({100 * s / max(tot_s, 1):4.1f}%) inst {inst[loc]:9d}  "
              f"{text[:60]:60s} | {reasons}")


if __name__ == "__main__":
    main()
