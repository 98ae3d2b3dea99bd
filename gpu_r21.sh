python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo "bench rc $?"; tail -3 gpurun_out/bench21.err
