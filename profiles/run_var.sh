# compare the default library with variant libraries: run_var.sh v1 v2 ...
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2402_14808_b200/librelay_b200_$v.so; fi
  [ -n "$SCALING" ] && RB_LIB=$L python profiles/diag_ctx_scaling.py 32 52 64,128,512 2>&1 | grep -v floor
  RB_LIB=$L python profiles/diag_c2.py 512,2048,8192
done
