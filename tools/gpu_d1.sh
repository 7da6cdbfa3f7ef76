# synthetic dataset (1) (b = 1024, a = 256, n = 32..512) strong-scaling
# efficiency at P = 2/4/8 from the per-rank step model (Fig. 3b shape), + flop-model ceiling
mkdir -p gpurun_out/d1
for n in 32 64 128 256 512; do
  timeout 900 python tools/scaling_sim.py D1 2,4,8 --no-seq --shape $n,1024,256 --strong --reps 1 > gpurun_out/d1/d1_n$n.txt 2>&1; echo n$n=$?
done
grep -h '"P"' gpurun_out/d1/*.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'T_ms' in d: print(d['n'], d['P'], d['Q'], d['T_ms'], d['E_strong'], d['E_flop_model'])"
