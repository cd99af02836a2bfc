mkdir -p gpurun_out
python -m pytest tests/test_gpu_dropin_cpp.py -x -q > gpurun_out/r2b_dropin.log 2>&1; echo rc=$? >> gpurun_out/r2b_dropin.log
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "not s26" > gpurun_out/r2b_parity.log 2>&1; echo rc=$? >> gpurun_out/r2b_parity.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode > gpurun_out/r2b_bench.log 2>&1; echo rc=$? >> gpurun_out/r2b_bench.log
timeout 1500 python -m pytest tests/test_gpu_acceptance.py -x -q -s > gpurun_out/r2b_accept.log 2>&1; echo rc=$? >> gpurun_out/r2b_accept.log
