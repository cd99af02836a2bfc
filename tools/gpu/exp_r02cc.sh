timeout 1500 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/lprol/libetbfs_b200.so" > gpurun_out/ab26cc.log 2>&1
timeout 900 python tools/ab_env.py --scale 28 --steps 2 --repeat 1 --variants "ETB_BASE=1" "ETB_LIB=tools/variants/lprol/libetbfs_b200.so" > gpurun_out/ab28cc.log 2>&1
cat gpurun_out/ab26cc.log gpurun_out/ab28cc.log
