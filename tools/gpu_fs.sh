mkdir -p gpurun_out/fs
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k distributed > gpurun_out/fs/fs.txt 2>&1; echo fs=$?
tail -15 gpurun_out/fs/fs.txt
