# end-rank ratio r (serinv_plan_ends) on the step model
mkdir -p gpurun_out/r
for r in 1.2 1.4; do timeout 600 python tools/scaling_sim.py C2 8 --reps 1 --r $r > gpurun_out/r/C2_r$r.txt 2>&1; echo C2 $r=$?; done
for r in 1.6 2.0; do timeout 900 python tools/scaling_sim.py C3 8 --strong --reps 1 --r $r > gpurun_out/r/C3_r$r.txt 2>&1; echo C3 $r=$?; done
for r in 1.2; do timeout 600 python tools/scaling_sim.py C4 8 --no-seq --reps 1 --r $r > gpurun_out/r/C4_r$r.txt 2>&1; echo C4 $r=$?; done
for f in gpurun_out/r/*.txt; do echo $f; grep -h '"P"' $f | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'T_ms' in d: print(d['n'], d['P'], d['Q'], d['T_ms'], d.get('E_weak', d.get('E_strong')), d['ppobtaf_ms'], d['ppobtasi_ms'])"; done
