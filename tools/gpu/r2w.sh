mkdir -p gpurun_out
timeout 600 python tools/c7_probe.py > gpurun_out/r2w_c7.log 2>&1
ETB_TD_AS_BU=0 timeout 600 python tools/c7_probe.py >> gpurun_out/r2w_c7.log 2>&1
timeout 900 python -m pytest tests/test_gpu_io.py tests/test_gpu_work.py -x -q > gpurun_out/r2w_tests.log 2>&1; echo rc=$? >> gpurun_out/r2w_tests.log
