timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validate.py tests/test_gpu_partition.py -x -q > gpurun_out/t_v.log 2>&1; tail -1 gpurun_out/t_v.log
timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/rowspair/libetbfs_b200.so" > gpurun_out/ab26v.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/rowspair/libetbfs_b200.so" > gpurun_out/ab22v.log 2>&1
cat gpurun_out/ab26v.log gpurun_out/ab22v.log
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 4 --cold --diag > gpurun_out/diag26_v.log 2>&1
