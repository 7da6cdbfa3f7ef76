timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q > gpurun_out/pytest_p.log 2>&1; echo tests=$?; tail -2 gpurun_out/pytest_p.log
for c in "C2 1" "C4 auto" "C5 auto" "C3 1"; do timeout 200 python tools/time1.py $c 2 2>&1 | tail -1; done > gpurun_out/sweep20.txt
cat gpurun_out/sweep20.txt
timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2.txt 2>&1; sed -n '/timeline/,$p' gpurun_out/crit_C2.txt
