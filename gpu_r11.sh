python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python profiles/diag_step_timeline.py 8192 2 0 60 2>&1 | tail -19
timeout 300 python profiles/diag_step_timeline.py 8192 3 0 60 2>&1 | tail -19
timeout 600 python -m pytest tests/test_relay_step.py -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo "bench rc $?"; tail -3 gpurun_out/bench11.err
