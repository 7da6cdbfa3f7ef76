# GPU parity (incl. Q sub-partitions) + multi-GPU step model with Q
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q/gpu_tests.txt 2>&1; echo tests=$?
tail -3 gpurun_out/q/gpu_tests.txt
timeout 900 python tools/scaling_sim.py C4 2,4,8 --q auto,2,8 > gpurun_out/q/scale_C4.txt 2>&1; echo simC4=$?
timeout 900 python tools/scaling_sim.py C2 2,4,8 --q 1,2 > gpurun_out/q/scale_C2.txt 2>&1; echo simC2=$?
timeout 1200 python tools/scaling_sim.py C5 2,8 --q auto > gpurun_out/q/scale_C5.txt 2>&1; echo simC5=$?
timeout 900 python tools/scaling_sim.py C3 8 --strong --q 1,2 > gpurun_out/q/scale_C3.txt 2>&1; echo simC3=$?
tail -n 12 gpurun_out/q/scale_*.txt
