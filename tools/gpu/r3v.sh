mkdir -p gpurun_out/r3v
ETB_LIB=tools/variants/checked/libetbfs_b200.so ETB_BFS_BLOCK=1024 ETB_SPLIT_RATIO=0.05 ETB_SPLIT_DIV=16 timeout 1500 python tools/checked_run.py > gpurun_out/r3v/checked_split_a.log 2>&1; echo rc=$? >> gpurun_out/r3v/checked_split_a.log
ETB_LIB=tools/variants/checked/libetbfs_b200.so ETB_BFS_BLOCK=1024 ETB_SPLIT_RATIO=0.05 ETB_SPLIT_TDW=16 timeout 1500 python tools/checked_run.py > gpurun_out/r3v/checked_split_b.log 2>&1; echo rc=$? >> gpurun_out/r3v/checked_split_b.log
ETB_LIB=tools/variants/checked/libetbfs_b200.so ETB_BFS_BLOCK=1024 ETB_SPLIT_RATIO=0.05 timeout 900 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_stress.py -m gpu -q > gpurun_out/r3v/checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r3v/checked_tests.log
