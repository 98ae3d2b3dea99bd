# One GPU round of evidence (run under gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash profiles/run_round.sh r01c'
# Writes everything under gpurun_out/<tag>_*; profiles/summarize_ncu.py turns
# the ncu reports into profiles/ncu_summary.json.
tag=${1:-run}
out=gpurun_out
mkdir -p $out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -15 | tee $out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee $out/${tag}_smoke.txt
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err; echo "ref rc $?"
timeout 900 python profiles/bench_configs.py --naive > $out/${tag}_configs.log 2>&1; echo "configs rc $?"
# launch list of the bench step (kernels of this repo only; cold-cache, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sys_attn|ctx_|kv_append" -c 60 --csv --log-file $out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 1 --sweep "" --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1; echo "ncu launches rc $?"
# one full capture of each kernel of the relay step at C2 s=8192
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sys_attn|ctx_" -c 2 -f \
  -o $out/${tag}_prof_step python profiles/diag_relay_timeline.py 8192 3 > $out/${tag}_ncu_step.log 2>&1; echo "ncu step rc $?"
# one full capture of the GQA-large system kernel (C4 shape, alone on all SMs)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sys_gqa -s 3 -c 1 -f \
  -o $out/${tag}_prof_gqa python profiles/diag_gqa_sys.py > $out/${tag}_ncu_gqa.log 2>&1; echo "ncu gqa rc $?"
