mkdir -p gpurun_out/r3q
ETB_SPLIT_TDW=16 timeout 1200 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_stress.py -m gpu -q > gpurun_out/r3q/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3q/pytest.log
timeout 2400 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_SPLIT_TDW=0" "ETB_SPLIT_TDW=8" "ETB_SPLIT_TDW=16" "ETB_SPLIT_TDW=24" "ETB_SPLIT_TDW=32" "ETB_SPLIT_TDW=16 ETB_SPLIT_DIV=2048" "ETB_SPLIT_TDW=16 ETB_SPLIT_RATIO=1.5" > gpurun_out/r3q/ab26.log 2>&1
timeout 2400 python tools/ab_env.py --scale 28 --repeat 1 --variants "ETB_SPLIT_TDW=0" "ETB_SPLIT_TDW=16" "ETB_SPLIT_TDW=32" > gpurun_out/r3q/ab28.log 2>&1
