"""Markdown error table from a GPU parity log (RB_PARITY_LOG jsonl written by
tests/gpu_util.py during `pytest -m gpu`).

    python profiles/parity_table.py profiles/r02/parity_<tag>.jsonl
"""
import json
import sys


def fmt(x):
    return f"{x:.2e}" if isinstance(x, float) else str(x)


def main():
    rows = [json.loads(l) for l in open(sys.argv[1])]
    print("| case | o max-abs | o rel (L2) | LSE max-abs | notes |")
    print("|---|---|---|---|---|")
    for r in rows:
        if r.get("kind") not in ("config", "suite", "integration"):
            continue
        notes = []
        for k in ("plan", "grid", "pairs", "cases", "naive_o_max_abs", "brute_force_max_abs",
                  "logit_max_rel", "token_streams_identical", "sampled_layers"):
            if k in r:
                v = r[k]
                if k == "plan":
                    v = f"nq={v['nq']} n_qt={v['n_qt']} grid={v['grid']} rr={v['rr']}"
                notes.append(f"{k}: {fmt(v)}")
        print(f"| {r['case']} | {fmt(r.get('o_max_abs', '-'))} | {fmt(r.get('o_rel', '-'))} | "
              f"{fmt(r.get('lse_max_abs', '-'))} | {'; '.join(notes)} |")
    # prefix-grouped element-wise cases (prefill, engine steps): worst per group
    groups = {}
    for r in rows:
        if r.get("kind") not in ("out", "lse"):
            continue
        for pre, name in (("prefill", "GPU system-KV prefill (SystemKvCache.prefill)"),
                          ("engine relay", "B200 engine steps, relay mode"),
                          ("engine baseline", "B200 engine steps, baseline mode"),
                          ("relay step over a prefilled", "relay step over a prefilled cache")):
            if r["case"].startswith(pre):
                g = groups.setdefault(name, {"out": 0.0, "rel": 0.0, "lse": 0.0, "n": 0})
                g["n"] += 1
                if r["kind"] == "out":
                    g["out"] = max(g["out"], r["max_abs"])
                    g["rel"] = max(g["rel"], r.get("rel", 0.0))
                else:
                    g["lse"] = max(g["lse"], r["max_abs"])
    for name, g in groups.items():
        print(f"| {name} | {fmt(g['out'])} | {fmt(g['rel'])} | {fmt(g['lse'])} | comparisons: {g['n']} |")
    eng = [r for r in rows if r.get("kind") == "engine"]
    if eng:
        print()
        print("Reference scheduler (`run_batch_job`) on the B200 engine, measured step costs:")
        print()
        print("| s | mode | simulated time (ms) | tokens/s | batch sizes |")
        print("|---|---|---|---|---|")
        for r in eng:
            print(f"| {r.get('s', '-')} | {r.get('mode', '-')} | {r['total_time_s'] * 1e3:.2f} | "
                  f"{r['tokens_per_s']:.0f} | {r['batch_hist']} |")
    print()
    print(f"Element-wise comparisons logged: {sum(1 for r in rows if r.get('kind') in ('out', 'lse'))} "
          f"(max over them: o {max([r['max_abs'] for r in rows if r.get('kind') == 'out'] or [0]):.2e}, "
          f"lse {max([r['max_abs'] for r in rows if r.get('kind') == 'lse'] or [0]):.2e}).")


if __name__ == "__main__":
    main()
