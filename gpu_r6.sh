python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -30
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc $?"; tail -3 gpurun_out/bench6.err
timeout 600 python profiles/bench_configs.py 2>&1 | tee gpurun_out/bench_configs6.txt
