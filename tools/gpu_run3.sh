set -x
./tools/mainloop_ubench > gpurun_out/mainloop_ubench.txt 2>&1
python tools/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1
python tools/trace.py selinv 128 1024 64 > gpurun_out/trace_C2_tw.txt 2>&1
SERINV_OPT=twist_min_n=0 python tools/trace.py selinv 365 2048 4 > gpurun_out/trace_C3_1s.txt 2>&1
python tools/trace.py selinv 365 2048 4 > gpurun_out/trace_C3_tw.txt 2>&1
