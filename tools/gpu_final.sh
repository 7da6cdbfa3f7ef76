mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/final/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
for c in C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo $c=$?
done
cat gpurun_out/final/bench_*.json
bash tools/ncu_run.sh C3
mv gpurun_out/ncu_C3 gpurun_out/final/ 2>/dev/null
