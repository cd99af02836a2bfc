timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py -x -q > gpurun_out/t_x.log 2>&1; tail -1 gpurun_out/t_x.log
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 1 --parts 8 --variants "ETB_BASE=1" > gpurun_out/ab22x_8.log 2>&1
timeout 900 python tools/ab_env.py --scale 26 --steps 3 --repeat 1 --parts 2 --variants "ETB_BASE=1" > gpurun_out/ab26x_2.log 2>&1
timeout 900 python tools/ab_env.py --scale 26 --steps 3 --repeat 1 --variants "ETB_BASE=1" > gpurun_out/ab26x_1.log 2>&1
cat gpurun_out/ab22x_8.log gpurun_out/ab26x_2.log gpurun_out/ab26x_1.log
ETB_LIB=tools/variants/checked/libetbfs_b200.so timeout 1500 python tools/checked_run.py > gpurun_out/checked_run.log 2>&1; echo rc=$? >> gpurun_out/checked_run.log; tail -5 gpurun_out/checked_run.log
