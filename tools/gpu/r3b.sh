mkdir -p gpurun_out/r3b
timeout 900 python -m pytest tests/test_gpu_download.py tests/test_capi.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r3b/pytest.log 2>&1; echo rc=$? >> gpurun_out/r3b/pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --secondary "22/16,28/16" --no-paper-mode --emulate-partitions "" > gpurun_out/r3b/bench.json 2> gpurun_out/r3b/bench.err; echo rc=$? >> gpurun_out/r3b/bench.err
nproc > gpurun_out/r3b/nproc.txt; free -g >> gpurun_out/r3b/nproc.txt; lscpu | head -20 >> gpurun_out/r3b/nproc.txt
