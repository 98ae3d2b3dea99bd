set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ls paper_2402_14808_b200/*.so oracle/*.so oracle/_ref
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sys_attn -s 3 -c 1 -o gpurun_out/prof_sys python bench.py --steps 3 --warmup 1 --sweep "" --no-cpu-baseline > gpurun_out/ncu_sys.log 2>&1; echo "ncu sys rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctx_attn -s 3 -c 1 -o gpurun_out/prof_ctx python bench.py --steps 3 --warmup 1 --sweep "" --no-cpu-baseline > gpurun_out/ncu_ctx.log 2>&1; echo "ncu ctx rc $?"
