# GPU parity run: every -m gpu test, per-case errors appended to
# gpurun_out/<tag>_parity.jsonl (tests/gpu_util.py), then the bench line.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash profiles/run_tests.sh r02a'
tag=${1:-run}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
rm -f $out/${tag}_parity.jsonl
RB_PARITY_LOG=$out/${tag}_parity.jsonl timeout 1500 python -m pytest tests/ -m gpu -q -rf -p no:cacheprovider ${PYTEST_ARGS} > $out/${tag}_pytest_full.txt 2>&1
tail -40 $out/${tag}_pytest_full.txt | tee $out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee $out/${tag}_smoke.txt
if [ "${2:-bench}" = "bench" ]; then
  timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
  tail -c 3000 $out/${tag}_bench.json
fi
