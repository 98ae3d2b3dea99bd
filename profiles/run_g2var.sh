# 256-row GQA kernel variants: per-tile timeline (CTA 0) + C4/C5 step times
# usage: bash profiles/run_g2var.sh v1 v2 ...  (librelay_b200_<v>.so, diag builds)
for v in "$@"; do
  echo "== $v"
  RB_LIB=paper_2402_14808_b200/librelay_b200_$v.so ROWS=4 timeout 120 python profiles/diag_gqa2_timeline.py 2>&1 | tail -8
done
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  echo "== $v"
  RB_LIB=$L timeout 300 python profiles/bench_configs.py --configs c4,c5 --steps 10 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], round(d['us_per_step'], 1), round(d['frac_of_roofline'], 3))"
done
