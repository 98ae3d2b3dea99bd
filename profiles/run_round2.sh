# Round-2 evidence run (under gpurun, one GPU):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash profiles/run_round2.sh r02m'
# Writes gpurun_out/<tag>_*; profiles/summarize_ncu.py turns the reports into
# profiles/ncu_summary.json.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee $out/${tag}_gpu.txt
RB_PARITY_LOG=$out/${tag}_parity.jsonl timeout 1500 python -m pytest tests/ -m gpu -q 2>&1 | tail -15 | tee $out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee $out/${tag}_smoke.txt
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err; echo "ref rc $?"
timeout 900 python profiles/bench_configs.py --naive > $out/${tag}_configs.log 2>&1; echo "configs rc $?"
cp $out/bench_configs.json $out/${tag}_bench_configs.json 2>/dev/null
# launch list of the bench step (this repo's kernels; cold-cache, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sys_attn|sys_gqa|ctx_|kv_append|rope_append" -c 80 --csv --log-file $out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 1 --sweep "" --configs "" --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1; echo "launches rc $?"
# full captures: the relay step's two kernels at C2 s=8192, the context kernel alone,
# the 256-row GQA system kernel alone at C4 and C5 shapes
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sys_attn|ctx_" -s 4 -c 2 -f \
  -o $out/${tag}_prof_step python profiles/diag_relay_timeline.py 8192 3 > $out/${tag}_ncu_step.log 2>&1; echo "step rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_ -s 6 -c 1 -f \
  -o $out/${tag}_prof_ctx python profiles/diag_ctx.py 32 52 128 3 > $out/${tag}_ncu_ctx.log 2>&1; echo "ctx rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sys_gqa2 -s 2 -c 1 -f \
  -o $out/${tag}_prof_gqa2 python profiles/diag_gqa_sys.py > $out/${tag}_ncu_gqa2.log 2>&1; echo "gqa2 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sys_gqa2 -s 2 -c 1 -f \
  -o $out/${tag}_prof_gqa2_c5 python profiles/diag_gqa_sys.py 256 64 8 65536 > $out/${tag}_ncu_gqa2_c5.log 2>&1; echo "gqa2 c5 rc $?"
