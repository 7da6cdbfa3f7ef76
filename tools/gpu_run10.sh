timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_parity.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; cat gpurun_out/bench_C2.json
