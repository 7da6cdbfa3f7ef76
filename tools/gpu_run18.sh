for o in "" "twist_max_b=4096" "twist_max_b=4096,si_split=0"; do SERINV_OPT="$o" timeout 200 python tools/time1.py C3 1 2 2>&1 | tail -1; done > gpurun_out/sweep18.txt
SERINV_OPT="twist_max_b=4096" timeout 300 python tools/trace.py selinv 96 2048 4 > gpurun_out/trace_C3s_tw.txt 2>&1
timeout 300 python tools/trace.py selinv 96 2048 4 > gpurun_out/trace_C3s_1s.txt 2>&1
cat gpurun_out/sweep18.txt; grep -E "makespan|utilisation|dip|POTRF end|running" gpurun_out/trace_C3s_tw.txt gpurun_out/trace_C3s_1s.txt
