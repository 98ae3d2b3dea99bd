for v in g2d g2nosm g2nomma; do
  echo "== $v"
  RB_LIB=paper_2402_14808_b200/librelay_b200_$v.so ROWS=2 timeout 120 python profiles/diag_gqa2_timeline.py 2>&1 | grep -v "^ *[0-9]\|^tile"
done
