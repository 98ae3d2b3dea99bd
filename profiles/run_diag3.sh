out=gpurun_out; mkdir -p $out
for s in 512 2048; do timeout 120 python profiles/diag_relay_timeline.py $s 3; done 2>&1 | grep -v "^    sm" | tee $out/d3_timeline.txt
timeout 120 python profiles/diag_relay_timeline.py 512 2 2>&1 | grep -v "^    sm" | tee $out/d3_timeline_ctx.txt
