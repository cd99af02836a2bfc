timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validate.py -x -q > gpurun_out/t_kk.log 2>&1; tail -1 gpurun_out/t_kk.log
timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/oldbar/libetbfs_b200.so" > gpurun_out/ab26kk.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/oldbar/libetbfs_b200.so" > gpurun_out/ab22kk.log 2>&1
cat gpurun_out/ab26kk.log gpurun_out/ab22kk.log
