mkdir -p gpurun_out/r3c
timeout 900 python -m pytest tests/test_gpu_download.py -m gpu -q > gpurun_out/r3c/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3c/pytest.log
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_X=0" "ETB_LIB=tools/variants/noda/libetbfs_b200.so" > gpurun_out/r3c/ab26.log 2>&1
