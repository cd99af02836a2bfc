mkdir -p gpurun_out
export ETB_LIB=tools/variants/checked/libetbfs_b200.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_partition.py tests/test_gpu_large_kernel.py -x -q > gpurun_out/r2p_checked.log 2>&1; echo rc=$? >> gpurun_out/r2p_checked.log
timeout 900 python tools/sanitize_run.py >> gpurun_out/r2p_checked.log 2>&1; echo rc=$? >> gpurun_out/r2p_checked.log
unset ETB_LIB
timeout 900 python tools/part_balance.py --scale 26 --parts 1,2,8 --roots 2 > gpurun_out/r2p_bal.log 2>&1
