# A/B of variant libraries on one box: C4/C5 relay steps (bench_configs), alternating
# usage: bash profiles/run_ab.sh "c4,c5" v1 v2 ...   (default = the production library)
CFG=$1; shift
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  RB_LIB=$L timeout 300 python profiles/bench_configs.py --configs $CFG --steps 10 2>&1 | grep "^{" | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$v', d['config'], round(d['us_per_step'], 1), round(d['frac_of_roofline'], 3), 'sys', round(d.get('sys_kernel_us', 0), 1))"
done
done
