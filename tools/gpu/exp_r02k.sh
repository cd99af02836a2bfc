ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 4 --cold --diag > gpurun_out/diag26_k1.log 2>&1
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 4 --cold --diag --parts 2 > gpurun_out/diag26_k2.log 2>&1
timeout 600 python tools/part_balance.py --scale 26 --parts 1,2 --roots 2 > gpurun_out/partbal26.log 2>&1
