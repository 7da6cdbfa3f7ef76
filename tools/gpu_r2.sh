mkdir -p gpurun_out/r2
timeout 600 python tools/scaling_sim.py C3 8 --strong --reps 1 --r 2.5 > gpurun_out/r2/C3_r2.5.txt 2>&1; echo C3=$?
timeout 600 python tools/scaling_sim.py C2 4 --reps 1 --r 1.2 > gpurun_out/r2/C2_P4_r1.2.txt 2>&1; echo C2=$?
for f in gpurun_out/r2/*.txt; do echo $f; grep -h '"P"' $f | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'T_ms' in d: print(d['n'], d['P'], d['Q'], d['T_ms'], d.get('E_weak', d.get('E_strong')))"; done
