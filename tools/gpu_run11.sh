timeout 900 python -m pytest tests/test_gpu_partitioned.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_part.log 2>&1; echo part=$?; tail -5 gpurun_out/pytest_part.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; cat gpurun_out/bench_C2.json
for o in "" "twist_last=0"; do
  for c in "C4 auto" "C4 8" "C4 4" "C5 auto" ; do SERINV_OPT="$o" timeout 120 python tools/time1.py $c 2 2>&1 | tail -1; done
done > gpurun_out/sweep11.txt
cat gpurun_out/sweep11.txt
