SERINV_OPT="fuse_trsm=1,split_chain=0" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo fused_tests=$?; tail -2 gpurun_out/pytest_fused.log
for o in "" "fuse_trsm=1,split_chain=0" "fuse_trsm=1,split_chain=0,update_group=2"; do
 for c in "C2 1" "C4 auto" "C5 auto" "C3 1"; do SERINV_OPT="$o" timeout 120 python tools/time1.py $c 2 2>&1 | tail -1; done
done > gpurun_out/sweep17.txt
SERINV_OPT="fuse_trsm=1,split_chain=0" timeout 300 python tools/critpath.py selinv 128 1024 64 > gpurun_out/crit_C2_fused.txt 2>&1
cat gpurun_out/sweep17.txt gpurun_out/crit_C2_fused.txt
