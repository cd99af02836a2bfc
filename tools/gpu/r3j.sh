mkdir -p gpurun_out/r3j
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_X=0" "ETB_LIB=tools/variants/lean/libetbfs_b200.so" > gpurun_out/r3j/ab26.log 2>&1
