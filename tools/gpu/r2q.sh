mkdir -p gpurun_out
ETB_LIB=tools/variants/checked/libetbfs_b200.so timeout 1500 python tools/checked_run.py > gpurun_out/r2q_checked.log 2>&1; echo rc=$? >> gpurun_out/r2q_checked.log
ETB_LIB=tools/variants/checked/libetbfs_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_partition.py tests/test_gpu_large_kernel.py -x -q > gpurun_out/r2q_checked_tests.log 2>&1; echo rc=$? >> gpurun_out/r2q_checked_tests.log
s=$SECONDS; timeout 1800 python bench.py > gpurun_out/r2n_bench.log 2> gpurun_out/r2n_bench.err; echo rc=$? wall=$((SECONDS-s)) >> gpurun_out/r2n_bench.log
s=$SECONDS; timeout 1800 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2n_ref.log 2> gpurun_out/r2n_ref.err; echo rc=$? wall=$((SECONDS-s)) >> gpurun_out/r2n_ref.log
