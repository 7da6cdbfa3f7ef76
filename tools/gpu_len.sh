# reduced-system nesting (dist_len) sweep at P = 8 on the step model
mkdir -p gpurun_out/len
for L in 0 8 4; do SERINV_OPT=dist_len=$L timeout 600 python tools/scaling_sim.py C2 8 --reps 1 > gpurun_out/len/C2_len$L.txt 2>&1; echo C2 $L=$?; done
for L in 0 16 8; do SERINV_OPT=dist_len=$L timeout 600 python tools/scaling_sim.py C4 8 --reps 1 > gpurun_out/len/C4_len$L.txt 2>&1; echo C4 $L=$?; done
for L in 0 128 32; do SERINV_OPT=dist_len=$L timeout 900 python tools/scaling_sim.py C5 8 --reps 1 > gpurun_out/len/C5_len$L.txt 2>&1; echo C5 $L=$?; done
grep -h '"P": 8' gpurun_out/len/*.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['Q'], d['T_ms'], d.get('E_weak'), max(d['ppobtaf_ms']), max(d['ppobtasi_ms']))"
