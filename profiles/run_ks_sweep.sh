for v in default ks3 ks4; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  echo "== $v"
  RB_LIB=$L SWEEP_GRIDS=24,29,34,40,46,52,60,68,76,84,90 python profiles/sweep_split.py 1024 2048 4096 8192
done
