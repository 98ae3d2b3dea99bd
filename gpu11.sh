python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5
timeout 300 python profiles/diag_e2e.py 2>&1 | tee gpurun_out/diag_e2e2.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err; echo "bench rc $?"; tail -3 gpurun_out/bench_r01i.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctx_attn -s 3 -c 1 -o gpurun_out/prof_ctx_r01i python bench.py --steps 3 --warmup 1 --sweep "" --no-cpu-baseline > gpurun_out/ncu_ctx.log 2>&1; echo "ncu rc $?"
