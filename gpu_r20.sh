cd paper_2402_14808_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DRB_STEP_TRACE=1 -I ../../include -c relay_step_sm100.cu -o ../build/relay_step_sm100.o && cd ../.. && nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2402_14808_b200/librelay_b200.so paper_2402_14808_b200/build/relay_step_sm100.o paper_2402_14808_b200/build/aux_kernels.o paper_2402_14808_b200/build/probe_sm100.o paper_2402_14808_b200/build/capi.o
true
timeout 300 python profiles/diag_softmax_trace.py 8192 1 60 2>&1 | tail -14
