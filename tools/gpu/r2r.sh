mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "BASE=1" "ETB_LIB=tools/variants/eager/libetbfs_b200.so" > gpurun_out/r2r_ab26.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --repeat 2 --variants "BASE=1" "ETB_LIB=tools/variants/eager/libetbfs_b200.so" > gpurun_out/r2r_ab22.log 2>&1
