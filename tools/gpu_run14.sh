python tools/gemm_phases.py > gpurun_out/gemm_phases.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/pytest_parity.log
for c in "C2 1" "C4 auto" "C5 auto" "C3 1"; do timeout 120 python tools/time1.py $c 2 2>&1 | tail -1; done > gpurun_out/sweep14.txt
cat gpurun_out/gemm_phases.txt gpurun_out/sweep14.txt
