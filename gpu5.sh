python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r01d.json 2> gpurun_out/bench_r01d.err; echo "bench rc $?"; tail -3 gpurun_out/bench_r01d.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sys_attn -s 3 -c 1 -o gpurun_out/prof_sys_r01d python bench.py --steps 3 --warmup 1 --sweep "" --no-cpu-baseline > gpurun_out/ncu_sys.log 2>&1; echo "ncu2 rc $?"
