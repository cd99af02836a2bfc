ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 2 --cold --diag > gpurun_out/d1.log 2>&1
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 2 --cold --diag --parts 2 > gpurun_out/d2.log 2>&1
timeout 600 python tools/block_balance.py --scale 26 --index 0 > gpurun_out/bb1.log 2>&1
