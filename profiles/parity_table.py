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
    print()
    print(f"Element-wise comparisons logged: {sum(1 for r in rows if r.get('kind') in ('out', 'lse'))} "
          f"(max over them: o {max([r['max_abs'] for r in rows if r.get('kind') == 'out'] or [0]):.2e}, "
          f"lse {max([r['max_abs'] for r in rows if r.get('kind') == 'lse'] or [0]):.2e}).")


if __name__ == "__main__":
    main()
