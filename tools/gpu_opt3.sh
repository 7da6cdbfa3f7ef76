# SERINV_OPT knob sweep on C3 (selinv, device time, best of 2)
mkdir -p gpurun_out/opt
for o in "" si_split=640 si_split=1024 si_split=0 update_group=2 update_group=8 wide_min_wave=0 wide_min_wave=1024 carry_chain=0 early_sig=0; do
  echo "== $o"; SERINV_OPT="$o" timeout 200 python tools/sweep.py C3:1 2>&1 | tail -1
done > gpurun_out/opt/C3_knobs.txt
cat gpurun_out/opt/C3_knobs.txt
