# ncu evidence of the round-2 kernels (run under gpurun; one GPU):
#   launch list of the bench step, --set full captures of the relay step's
#   two kernels (C2 s=8192), the context kernel alone, and the 256-row GQA
#   system kernel alone at C4.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sys_attn|sys_gqa|ctx_|kv_append" -c 80 --csv --log-file $out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 1 --sweep "" --configs "" --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1; echo "launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sys_attn|ctx_" -s 4 -c 2 -f \
  -o $out/${tag}_prof_step python profiles/diag_relay_timeline.py 8192 3 > $out/${tag}_ncu_step.log 2>&1; echo "step rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_ -s 6 -c 1 -f \
  -o $out/${tag}_prof_ctx python profiles/diag_ctx.py 32 52 128 3 > $out/${tag}_ncu_ctx.log 2>&1; echo "ctx rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sys_gqa2 -s 3 -c 1 -f \
  -o $out/${tag}_prof_gqa2 python profiles/diag_gqa_sys.py > $out/${tag}_ncu_gqa2.log 2>&1; echo "gqa2 rc $?"
