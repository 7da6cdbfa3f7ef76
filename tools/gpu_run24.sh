timeout 900 python -m pytest tests/test_gpu_partitioned.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_p.log 2>&1; echo tests=$?; tail -2 gpurun_out/pytest_p.log
for r in 1.0 1.3 1.7 2.2; do timeout 200 python tools/time1.py C4 4 2 $r 2>&1 | tail -1; timeout 200 python tools/time1.py C4 6 2 $r 2>&1 | tail -1; done > gpurun_out/sweep24.txt
for r in 1.0 1.5 2.0; do timeout 200 python tools/time1.py C5 256x8 2 $r 2>&1 | tail -1; done >> gpurun_out/sweep24.txt
cat gpurun_out/sweep24.txt
