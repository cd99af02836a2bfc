timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validate.py tests/test_gpu_stress.py tests/test_gpu_checks.py tests/test_gpu_dropin_cpp.py -x -q > gpurun_out/t_t.log 2>&1; tail -1 gpurun_out/t_t.log
timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/head/libetbfs_b200.so" > gpurun_out/ab26t.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/head/libetbfs_b200.so" > gpurun_out/ab22t.log 2>&1
timeout 900 python tools/ab_env.py --scale 24 --edgefactor 4 --steps 2 --repeat 1 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/head/libetbfs_b200.so" > gpurun_out/ab24t.log 2>&1
cat gpurun_out/ab26t.log gpurun_out/ab22t.log gpurun_out/ab24t.log
