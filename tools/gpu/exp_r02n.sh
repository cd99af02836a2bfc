timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/notma/libetbfs_b200.so" > gpurun_out/ab26n.log 2>&1
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/notma/libetbfs_b200.so" > gpurun_out/ab22n.log 2>&1
cat gpurun_out/ab26n.log gpurun_out/ab22n.log
