mkdir -p gpurun_out/r3k
ETB_SPLIT_RATIO=1.0 ETB_SPLIT_DIV=64 timeout 1200 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_stress.py -m gpu -q -x > gpurun_out/r3k/pytest_split.log 2>&1; echo rc=$? >> gpurun_out/r3k/pytest_split.log
timeout 2400 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_LIB=tools/variants/head/libetbfs_b200.so" "ETB_SPLIT_RATIO=0" "ETB_SPLIT_RATIO=1.5" "ETB_SPLIT_RATIO=2.5" "ETB_SPLIT_RATIO=1.5 ETB_SPLIT_DIV=256" "ETB_SPLIT_RATIO=1.5 ETB_SPLIT_DIV=4096" > gpurun_out/r3k/ab26.log 2>&1
