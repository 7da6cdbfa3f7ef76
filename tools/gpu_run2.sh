set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in C2 C4 C3; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --partitions 1 > gpurun_out/bench_${c}_tw.json 2> gpurun_out/bench_${c}_tw.err; echo $c=$?; cat gpurun_out/bench_${c}_tw.json
done
SERINV_OPT=twist_min_n=0 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e --partitions 1 > gpurun_out/bench_C4_1s.json; cat gpurun_out/bench_C4_1s.json
