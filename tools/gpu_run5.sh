./tools/tile_ubench > gpurun_out/tile_ubench.txt 2>&1
for o in "si_split=0" "si_split=0,twist_min_n=0" "si_split=160"; do
  SERINV_OPT="$o" timeout 120 python tools/time1.py C3 1 2 2>&1 | tail -1
done >> gpurun_out/sweep_C3.txt
for o in "si_split=0" "si_split=0,update_group=2" "si_split=0,update_group=3" "si_split=0,critical_queues=1,max_crit=64"; do
  SERINV_OPT="$o" timeout 120 python tools/time1.py C2 1 3 2>&1 | tail -1
  SERINV_OPT="$o" timeout 120 python tools/time1.py C4 1 3 2>&1 | tail -1
done >> gpurun_out/sweep_C2.txt
python tools/trace.py pselinv 16384 64 8 --P auto > gpurun_out/trace_C5.txt 2>&1
