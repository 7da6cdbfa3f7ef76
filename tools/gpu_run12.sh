for c in "C4 2" "C4 3" "C4 4" "C4 6" "C4 4x3" "C5 auto" "C5 128x8" "C5 256x16" "C5 512x16" "C5 256x8x4" "C5 128x16" "C5 512x32x4"; do timeout 120 python tools/time1.py $c 2 2>&1 | tail -1; done > gpurun_out/sweep12.txt
SERINV_OPT=twist_last=0 timeout 120 python tools/time1.py C4 4 2 2>&1 | tail -1 >> gpurun_out/sweep12.txt
cat gpurun_out/sweep12.txt
bash tools/ncu_run.sh C2
