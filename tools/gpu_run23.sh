timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu_tests=$?; tail -3 gpurun_out/pytest_gpu.log
for c in "C2 1" "C4 auto" "C5 auto" "C3 1"; do timeout 200 python tools/time1.py $c 2 2>&1 | tail -1; done > gpurun_out/sweep23.txt
cat gpurun_out/sweep23.txt
