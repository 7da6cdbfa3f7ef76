# twisted reduced solve: GPU parity, step model C2/C4 at P = 8, single-GPU C4/C5 bench
mkdir -p gpurun_out/tw
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tw/gpu_tests.txt 2>&1; echo tests=$?; tail -2 gpurun_out/tw/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tw/smoke.log 2>&1; echo smoke=$?
timeout 600 python tools/scaling_sim.py C2 2,4,8 --reps 1 > gpurun_out/tw/model_C2.txt 2>&1; echo simC2=$?
timeout 600 python tools/scaling_sim.py C4 2,4,8 --no-seq > gpurun_out/tw/model_C4.txt 2>&1; echo simC4=$?
SERINV_OPT=twist_reduced=0 timeout 600 python tools/scaling_sim.py C2 8 --reps 1 > gpurun_out/tw/model_C2_off.txt 2>&1; echo simC2off=$?
for c in C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/tw/bench_$c.json 2> gpurun_out/tw/bench_$c.err; echo $c=$?
done
grep -h '"P"' gpurun_out/tw/model_*.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'T_ms' in d: print(d['n'], d['P'], d['Q'], d['T_ms'], d.get('E_weak'), max(d['ppobtaf_ms']), max(d['ppobtasi_ms']))"
cat gpurun_out/tw/bench_*.json
