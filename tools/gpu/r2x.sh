mkdir -p gpurun_out
timeout 600 python tools/c7_probe.py > gpurun_out/r2x_c7.log 2>&1
for i in 1 2; do timeout 1500 python -m pytest tests/test_gpu_acceptance.py -x -q -s > gpurun_out/r2x_accept$i.log 2>&1; echo rc=$? >> gpurun_out/r2x_accept$i.log; done
