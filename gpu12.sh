python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5
timeout 300 python profiles/diag_sys_timeline.py 512 8192 2>&1 | tee gpurun_out/diag_timeline5.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r01j.json 2> gpurun_out/bench_r01j.err; echo "bench rc $?"; tail -3 gpurun_out/bench_r01j.err
