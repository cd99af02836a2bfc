timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -x -q > gpurun_out/t_g.log 2>&1; tail -1 gpurun_out/t_g.log
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 8 --cold --diag > gpurun_out/diag26_g.log 2>&1
timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/rowsold/libetbfs_b200.so" > gpurun_out/ab26g.log 2>&1
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/rowsold/libetbfs_b200.so" > gpurun_out/ab22g.log 2>&1
cat gpurun_out/ab26g.log gpurun_out/ab22g.log
