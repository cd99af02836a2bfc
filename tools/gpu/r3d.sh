mkdir -p gpurun_out/r3d
timeout 900 python -m pytest tests/test_gpu_download.py -m gpu -q > gpurun_out/r3d/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3d/pytest.log
timeout 900 python tools/root_profile.py --cold --scale 26 > gpurun_out/r3d/rp26.log 2>&1
