mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/r2u_part.log 2>&1; echo rc=$? >> gpurun_out/r2u_part.log
ETB_LIB=tools/variants/checked/libetbfs_b200.so timeout 1500 python tools/checked_run.py > gpurun_out/r2u_checked.log 2>&1; echo rc=$? >> gpurun_out/r2u_checked.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode > gpurun_out/r2u_bench.log 2>&1; echo rc=$? >> gpurun_out/r2u_bench.log
