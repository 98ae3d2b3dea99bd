python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python profiles/diag_step_timeline.py 8192 2 0 60 2>&1 | tail -30
