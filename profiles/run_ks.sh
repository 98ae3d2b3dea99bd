for v in default ks3 ks4; do
  if [ $v = default ]; then python profiles/diag_c2.py 512,2048,8192,32768; else RB_LIB=paper_2402_14808_b200/librelay_b200_$v.so python profiles/diag_c2.py 512,2048,8192,32768; fi
done
