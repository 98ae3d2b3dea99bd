python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python -m pytest tests/test_relay_step.py -m gpu -q -k "layouts" 2>&1 | tail -15
