timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_parity.log
timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2.txt 2>&1
timeout 300 python tools/trace.py selinv 128 1024 64 > gpurun_out/trace_C2.txt 2>&1
for o in "" "chol8=0"; do
  for c in C2 C4 C3; do SERINV_OPT="$o" timeout 120 python tools/time1.py $c 1 2 2>&1 | tail -1; done
done > gpurun_out/sweep8.txt
