for o in "" "chain_syrk=0" "chain_syrk=0,update_group=2" "update_group=2" "update_group=8" "si_split=0" "wide_min_wave=256" "wide_min_wave=1024"; do SERINV_OPT="$o" timeout 120 python tools/time1.py C2 1 3 2>&1 | tail -1; done > gpurun_out/sweep16.txt
for o in "" "chain_syrk=0" "update_group=2" "update_group=8"; do SERINV_OPT="$o" timeout 120 python tools/time1.py C4 auto 3 2>&1 | tail -1; done >> gpurun_out/sweep16.txt
cat gpurun_out/sweep16.txt
