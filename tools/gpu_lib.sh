# vendor-library comparator (tools/library_arm.py) on every config, plus our arm at C2
mkdir -p gpurun_out/lib
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lib/smoke.log 2>&1; echo smoke=$?
for c in C2 C4 C5 C3; do
  timeout 600 python bench.py --impl library --config $c --steps 3 --warmup 2 > gpurun_out/lib/lib_$c.json 2> gpurun_out/lib/lib_$c.err; echo lib$c=$?
done
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu > gpurun_out/lib/ours_C2.json 2> gpurun_out/lib/ours_C2.err; echo oursC2=$?
cat gpurun_out/lib/*.json
