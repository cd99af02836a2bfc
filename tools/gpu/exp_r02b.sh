set -x
./tests/cpp/bin/test_prims > gpurun_out/prims.log 2>&1; echo rc=$? >> gpurun_out/prims.log; tail -3 gpurun_out/prims.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q > gpurun_out/parity.log 2>&1; tail -3 gpurun_out/parity.log
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 26 --roots 8 --cold --diag > gpurun_out/diag26.log 2>&1
ETB_LIB=tools/variants/misscyc/libetbfs_b200.so timeout 600 python tools/root_profile.py --scale 22 --roots 8 --cold --diag > gpurun_out/diag22.log 2>&1
timeout 900 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" "ETB_LIB=tools/variants/noda/libetbfs_b200.so" > gpurun_out/ab26.log 2>&1
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" > gpurun_out/ab22.log 2>&1
cat gpurun_out/ab26.log gpurun_out/ab22.log
