python -m paper_2402_14808_b200.build 2>&1 | tail -1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python profiles/diag_step_timeline.py 8192 2 60 2>&1 | tail -17
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench18.json 2> gpurun_out/bench18.err; echo "bench rc $?"; tail -3 gpurun_out/bench18.err
