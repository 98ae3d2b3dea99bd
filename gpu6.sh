python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 300 python profiles/diag_sys_timeline.py 512 2048 8192 32768 2>&1 | tee gpurun_out/diag_timeline.txt
