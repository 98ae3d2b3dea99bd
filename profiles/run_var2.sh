# variants: C2 step at several s + the C3/C4 configs + context scaling
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  echo "== $v"
  RB_LIB=$L python profiles/diag_ctx_scaling.py 32 52 128,512 2>&1 | grep -v floor
  RB_LIB=$L python profiles/diag_c2.py 512,2048,4096,8192
  RB_LIB=$L python profiles/bench_configs.py --configs c3,c4 --steps 10 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], round(d['us_per_step'], 1), round(d['frac_of_roofline'], 3))"
done
