python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --steps 20 --sweep 512,2048,8192,32768 > gpurun_out/bench24.json 2> gpurun_out/bench24.err; echo "bench rc $?"; tail -3 gpurun_out/bench24.err
timeout 600 ncu --metrics sm__icc_request_hit_rate.pct,gpu__time_duration.sum,smsp__pcsamp_warps_issue_stalled_no_instructions --clock-control none -k regex:relay_step -s 1 -c 1 python profiles/repro_step.py 32 52 52 8192 128 0 16 1 2>&1 | grep -E "icc|duration|no_instr"
