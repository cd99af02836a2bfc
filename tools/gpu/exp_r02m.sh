ETB_LIB=tools/variants/checked/libetbfs_b200.so timeout 600 python tools/gpu/tma_check.py 26 > gpurun_out/tma_checked.log 2>&1
ETB_LIB=tools/variants/war/libetbfs_b200.so timeout 600 python tools/gpu/tma_check.py 26 > gpurun_out/tma_war.log 2>&1
tail -5 gpurun_out/tma_checked.log; tail -3 gpurun_out/tma_war.log
