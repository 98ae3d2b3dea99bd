python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/test_relay_step.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo "bench rc $?"; tail -3 gpurun_out/bench19.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:relay_step -s 1 -c 1 -o gpurun_out/prof_step19 python profiles/repro_step.py 32 52 52 8192 128 0 16 3 > gpurun_out/ncu_step.log 2>&1; echo "ncu rc $?"
