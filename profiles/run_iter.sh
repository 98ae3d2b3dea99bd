# quick iteration: GPU tests, context kernel scaling, bench line
out=gpurun_out; mkdir -p $out; tag=${1:-it}
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -15 | tee $out/${tag}_pytest.txt
timeout 300 python profiles/diag_ctx_scaling.py 32 52 64,128,256,512,1024 2>&1 | tee $out/${tag}_ctx_scaling.txt
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
