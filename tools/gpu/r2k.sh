mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/r2k_part.log 2>&1; echo rc=$? >> gpurun_out/r2k_part.log
timeout 900 python tools/part_balance.py --scale 26 --parts 1,2,4,8 --roots 3 > gpurun_out/r2k_bal.log 2>&1; echo rc=$? >> gpurun_out/r2k_bal.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode > gpurun_out/r2k_bench.log 2>&1; echo rc=$? >> gpurun_out/r2k_bench.log
