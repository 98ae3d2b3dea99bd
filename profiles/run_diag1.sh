out=gpurun_out; mkdir -p $out
timeout 300 python profiles/diag_ctx_scaling.py 32 52 64,128,256,512,1024 2>&1 | tee $out/d1_ctx_scaling.txt
RB_LIB=paper_2402_14808_b200/librelay_b200_nocomp.so timeout 300 python profiles/diag_ctx_scaling.py 32 52 64,128,256,512,1024 2>&1 | tee $out/d1_ctx_scaling_nocomp.txt
