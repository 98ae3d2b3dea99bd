out=gpurun_out; mkdir -p $out
for s in 512 2048 8192; do timeout 120 python profiles/diag_relay_timeline.py $s 3; done 2>&1 | tee $out/d2_timeline.txt
for s in 512 2048; do timeout 120 python profiles/diag_relay_timeline.py $s 1; done 2>&1 | tee $out/d2_timeline_sys.txt
