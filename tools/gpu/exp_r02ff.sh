timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validate.py tests/test_gpu_partition.py -x -q > gpurun_out/t_ff.log 2>&1; tail -1 gpurun_out/t_ff.log
timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/nothird/libetbfs_b200.so" > gpurun_out/ab26ff.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/nothird/libetbfs_b200.so" > gpurun_out/ab22ff.log 2>&1
timeout 900 python tools/ab_env.py --scale 28 --steps 2 --repeat 1 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/nothird/libetbfs_b200.so" > gpurun_out/ab28ff.log 2>&1
cat gpurun_out/ab26ff.log gpurun_out/ab22ff.log gpurun_out/ab28ff.log
