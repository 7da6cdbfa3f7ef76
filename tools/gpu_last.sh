mkdir -p gpurun_out/last
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/last/gpu_tests.txt 2>&1; echo tests=$?; tail -2 gpurun_out/last/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/last/smoke.log
timeout 600 python bench.py > gpurun_out/last/bench_default.json 2> gpurun_out/last/bench_default.err; echo bench=$?
cat gpurun_out/last/bench_default.json
