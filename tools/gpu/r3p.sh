mkdir -p gpurun_out/r3p
timeout 1200 python -m pytest tests/test_gpu_large_kernel.py -m gpu -q > gpurun_out/r3p/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3p/pytest.log
