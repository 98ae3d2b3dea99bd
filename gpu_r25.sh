python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k hsd 2>&1 | grep -E "Error|assert|max" | head -10
timeout 600 ncu --set full --clock-control none --import-source on -k regex:relay_step -s 1 -c 1 -o gpurun_out/prof_step25 python profiles/repro_step.py 32 52 52 8192 128 0 16 3 > gpurun_out/ncu_step.log 2>&1; echo "ncu rc $?"
