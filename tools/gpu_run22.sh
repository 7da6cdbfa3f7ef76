timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2.txt 2>&1
SERINV_OPT=twist_min_n=0 timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2_1s.txt 2>&1
cat gpurun_out/crit_C2.txt gpurun_out/crit_C2_1s.txt
