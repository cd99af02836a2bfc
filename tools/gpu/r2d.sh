mkdir -p gpurun_out
timeout 600 python tools/gpu/td_check.py 20 > gpurun_out/r2d_td.log 2>&1; echo rc=$? >> gpurun_out/r2d_td.log
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_part.log 2>&1; echo rc=$? >> gpurun_out/r2d_part.log
timeout 1500 python -m pytest tests/test_gpu_acceptance.py -x -q -s > gpurun_out/r2d_accept.log 2>&1; echo rc=$? >> gpurun_out/r2d_accept.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode > gpurun_out/r2d_bench.log 2>&1; echo rc=$? >> gpurun_out/r2d_bench.log
