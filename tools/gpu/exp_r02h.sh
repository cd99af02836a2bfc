timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_validate.py -x -q > gpurun_out/t_h.log 2>&1; tail -1 gpurun_out/t_h.log
timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/prev/libetbfs_b200.so" "ETB_L2_PERSIST=1" > gpurun_out/ab26h.log 2>&1
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/prev/libetbfs_b200.so" "ETB_L2_PERSIST=1" > gpurun_out/ab22h.log 2>&1
timeout 900 python tools/ab_env.py --scale 28 --steps 2 --repeat 1 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" > gpurun_out/ab28h.log 2>&1
cat gpurun_out/ab26h.log gpurun_out/ab22h.log gpurun_out/ab28h.log
