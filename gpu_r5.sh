python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 120 python profiles/repro_step.py 32 8 8 1000 128 2>&1 | tail -2
timeout 600 python -m pytest tests/test_relay_step.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -30
