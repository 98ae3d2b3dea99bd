python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | grep -E "passed|failed|Error|assert |max" | head -20
timeout 600 python bench.py --no-cpu-baseline --steps 20 --sweep 512,2048,8192,32768 > gpurun_out/bench27.json 2> gpurun_out/bench27.err; echo "bench rc $?"; tail -3 gpurun_out/bench27.err
