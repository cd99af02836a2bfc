timeout 2000 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/mf128/libetbfs_b200.so" "ETB_LIB=tools/variants/mf256/libetbfs_b200.so" "ETB_LIB=tools/variants/mf512/libetbfs_b200.so" > gpurun_out/ab26dd.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --steps 3 --repeat 1 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/mf128/libetbfs_b200.so" "ETB_LIB=tools/variants/mf256/libetbfs_b200.so" > gpurun_out/ab22dd.log 2>&1
cat gpurun_out/ab26dd.log gpurun_out/ab22dd.log
