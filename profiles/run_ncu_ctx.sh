out=gpurun_out; mkdir -p $out
tag=${1:-ctx}
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-max-passes 50 --warp-sampling-buffer-size 536870912 -k regex:ctx_ -s 6 -c 1 -f \
  -o $out/${tag}_prof_ctx python profiles/diag_ctx.py 32 52 128 3 > $out/${tag}_ncu_ctx.log 2>&1; echo "ctx rc $?"
