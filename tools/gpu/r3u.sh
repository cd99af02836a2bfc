mkdir -p gpurun_out/r3u
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3u/smoke.log 2>&1; echo rc=$? >> gpurun_out/r3u/smoke.log
timeout 1500 python -m pytest tests/test_gpu_large_kernel.py tests/test_gpu_parity_full.py tests/test_gpu_download.py -m gpu -q > gpurun_out/r3u/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3u/pytest.log
timeout 900 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_X=0" "ETB_SPLIT_RATIO=0" > gpurun_out/r3u/ab26.log 2>&1
