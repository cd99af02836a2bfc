mkdir -p gpurun_out/r3i
timeout 1200 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_stress.py -m gpu -q -x > gpurun_out/r3i/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3i/pytest.log
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_LIB=tools/variants/nosnap/libetbfs_b200.so" "ETB_X=1" "ETB_LIB=tools/variants/snap3/libetbfs_b200.so" > gpurun_out/r3i/ab26.log 2>&1
timeout 1800 python tools/ab_env.py --scale 28 --repeat 2 --variants "ETB_LIB=tools/variants/nosnap/libetbfs_b200.so" "ETB_X=1" "ETB_LIB=tools/variants/snap3/libetbfs_b200.so" > gpurun_out/r3i/ab28.log 2>&1
