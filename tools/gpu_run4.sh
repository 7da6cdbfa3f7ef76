./tools/leaf_ubench > gpurun_out/leaf_ubench.txt 2>&1
for o in "" "urgent_ctas=2" "urgent_ctas=4" "urgent_ctas=8" "rts1_chain=1" "update_group=2" "update_group=8" "si_split=0" "si_split=640" "fuse_trsm=1,split_chain=0" "fuse_trsm=1,fuse_trsm3=1,split_chain=0" "critical_queues=0" "twist_min_n=0"; do
  SERINV_OPT="$o" timeout 120 python tools/time1.py C2 1 3 2>&1 | tail -1
done >> gpurun_out/sweep_C2.txt
python tools/trace.py selinv 365 2048 4 > gpurun_out/trace_C3_tw2.txt 2>&1
python tools/trace.py selinv 16384 64 8 --P auto > gpurun_out/trace_C5.txt 2>&1
