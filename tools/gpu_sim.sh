# partition-plan sweep (one GPU) + multi-GPU step model from measured per-rank phases
mkdir -p gpurun_out/sim
timeout 900 python tools/sweep.py C5:auto,512x16,1024x32,2048x64x4,128x8,1024x16x2,4096x128x4 > gpurun_out/sim/sweep_C5.txt 2>&1; echo sweepC5=$?
timeout 600 python tools/sweep.py C4:auto,1,2,3,4,6,8 C2:1,2,3 > gpurun_out/sim/sweep_C4C2.txt 2>&1; echo sweepC4=$?
timeout 900 python tools/scaling_sim.py C4 1,2,4,8 > gpurun_out/sim/scale_C4.txt 2>&1; echo simC4=$?
timeout 900 python tools/scaling_sim.py C5 1,2,4,8 > gpurun_out/sim/scale_C5.txt 2>&1; echo simC5=$?
timeout 900 python tools/scaling_sim.py C3 1,8 --strong > gpurun_out/sim/scale_C3.txt 2>&1; echo simC3=$?
tail -n 30 gpurun_out/sim/*.txt
