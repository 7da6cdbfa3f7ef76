timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2.txt 2>&1
for c in "C2 1" "C4 auto" "C5 auto" "C3 1"; do timeout 120 python tools/time1.py $c 2 2>&1 | tail -1; done > gpurun_out/sweep15.txt
SERINV_OPT=early_sig=0 timeout 120 python tools/time1.py C2 1 2 2>&1 | tail -1 >> gpurun_out/sweep15.txt
cat gpurun_out/sweep15.txt gpurun_out/crit_C2.txt
