mkdir -p gpurun_out/r3m
timeout 900 python tools/root_profile.py --cold --scale 26 > gpurun_out/r3m/rp26.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3m/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r3m/pytest_gpu.log
