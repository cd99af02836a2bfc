timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/head/libetbfs_b200.so" > gpurun_out/ab26u.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/head/libetbfs_b200.so" > gpurun_out/ab22u.log 2>&1
cat gpurun_out/ab26u.log gpurun_out/ab22u.log
