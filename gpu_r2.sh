python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python profiles/diag_sys_timeline.py 512 8192 2>&1 | tee gpurun_out/diag_timeline.txt
DIAG_MODE=sys timeout 300 python profiles/diag_sys_timeline.py 8192 2>&1 | tee -a gpurun_out/diag_timeline.txt
timeout 600 python profiles/bench_configs.py --naive 2>&1 | tee gpurun_out/bench_configs.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|kv_append|fusion" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --sweep "" --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
