timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for o in "" "wide_min_wave=0" "si_split=0" "wide_min_wave=256" ; do
  SERINV_OPT="$o" timeout 120 python tools/time1.py C3 1 2 2>&1 | tail -1
  SERINV_OPT="$o" timeout 120 python tools/time1.py C2 1 3 2>&1 | tail -1
done > gpurun_out/sweep6.txt
python tools/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1
