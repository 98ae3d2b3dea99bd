python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 120 python profiles/repro_step.py 4 4 4 64 33 2>&1 | tail -2
timeout 120 python profiles/repro_step.py 32 8 8 1000 128 0 16 1 2>&1 | tail -2
timeout 120 python profiles/repro_step.py 32 8 8 1000 128 0 16 2 2>&1 | tail -2
timeout 120 python profiles/repro_step.py 16 8 8 1000 128 2>&1 | tail -2
timeout 120 python profiles/repro_step.py 32 8 8 128 128 2>&1 | tail -2
timeout 300 compute-sanitizer --tool memcheck python profiles/repro_step.py 32 8 8 1000 128 2>&1 | head -60
