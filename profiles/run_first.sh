tag=r02k
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
RB_PARITY_LOG=$out/${tag}_parity.jsonl timeout 1200 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -15 | tee $out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee $out/${tag}_smoke.txt
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
