ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 8 --cold --diag > gpurun_out/diag26_f.log 2>&1
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 22 --roots 4 --cold --diag > gpurun_out/diag22_f.log 2>&1
