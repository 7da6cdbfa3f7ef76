# end-of-round: smoke, bench lines (N = 1) for C2..C5, dataset (1) strong-scaling sweep
mkdir -p gpurun_out/final2
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/final2/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final2/gpu_tests.txt 2>&1; echo tests=$?; tail -2 gpurun_out/final2/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo smoke=$?
for c in C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final2/bench_$c.json 2> gpurun_out/final2/bench_$c.err; echo $c=$?
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final2/bench_reference_C2.json 2>&1; echo ref=$?
cat gpurun_out/final2/bench_*.json
bash tools/gpu_d1.sh
timeout 900 python tools/scaling_sim.py C4 2,4,8 --no-seq > gpurun_out/final2/model_C4.txt 2>&1; echo simC4=$?
timeout 1200 python tools/scaling_sim.py C5 2,4,8 --no-seq --reps 1 > gpurun_out/final2/model_C5.txt 2>&1; echo simC5=$?
tail -n 4 gpurun_out/final2/model_*.txt
