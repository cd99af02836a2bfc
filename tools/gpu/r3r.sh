mkdir -p gpurun_out/r3r
ETB_SPLIT_TDW=64 timeout 1200 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_stress.py -m gpu -q > gpurun_out/r3r/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3r/pytest.log
timeout 2400 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_SPLIT_TDW=0" "ETB_SPLIT_TDW=64" "ETB_SPLIT_TDW=16" > gpurun_out/r3r/ab26.log 2>&1
timeout 2400 python tools/ab_env.py --scale 28 --repeat 1 --variants "ETB_SPLIT_TDW=0" "ETB_SPLIT_TDW=64" "ETB_SPLIT_TDW=8" > gpurun_out/r3r/ab28.log 2>&1
