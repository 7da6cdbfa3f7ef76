mkdir -p gpurun_out/opt
for o in "" update_group=3 update_group=5 update_group=6 wide_min_wave=384 wide_min_wave=768; do
  echo "== $o"; SERINV_OPT="$o" timeout 200 python tools/sweep.py C3:1 2>&1 | tail -1
done > gpurun_out/opt/C3_knobs2.txt
for o in "" update_group=3 update_group=5 update_group=6; do
  echo "== $o"; SERINV_OPT="$o" timeout 200 python tools/sweep.py C2:1 2>&1 | tail -1
done >> gpurun_out/opt/C3_knobs2.txt
cat gpurun_out/opt/C3_knobs2.txt
