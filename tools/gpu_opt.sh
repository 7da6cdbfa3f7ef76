# SERINV_OPT knob sweep on C2 (selinv, device time, best of 3)
mkdir -p gpurun_out/opt
for o in "" update_group=2 update_group=8 si_split=0 si_split=160 si_split=640 wide_min_wave=0 wide_min_wave=256 wide_min_wave=1024 urgent_ctas=2 urgent_ctas=4 carry_chain=0 "carry_min_b=1024" rts1_chain=1 fuse_trsm=1 early_sig=0; do
  echo "== $o"; SERINV_OPT="$o" timeout 120 python tools/sweep.py C2:1 2>&1 | tail -1
done > gpurun_out/opt/C2_knobs.txt
cat gpurun_out/opt/C2_knobs.txt
