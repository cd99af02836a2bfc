mkdir -p gpurun_out
timeout 600 python tools/gpu/td_check.py 20 > gpurun_out/r2c_td.log 2>&1; echo rc=$? >> gpurun_out/r2c_td.log
timeout 600 python -m pytest tests/test_gpu_dropin_cpp.py -x -q > gpurun_out/r2c_dropin.log 2>&1; echo rc=$? >> gpurun_out/r2c_dropin.log
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/r2c_part.log 2>&1; echo rc=$? >> gpurun_out/r2c_part.log
