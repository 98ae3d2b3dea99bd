# same-box A/B of library variants on the C2 step at several s (diag_c2.py)
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  echo "== $v"
  RB_LIB=$L timeout 300 python profiles/diag_c2.py 512,2048,4096,8192 2>&1 | tail -4
done
done
