nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dsmem_probe_bench.cu -o /tmp/dsmem.bin && timeout 120 /tmp/dsmem.bin > gpurun_out/dsmem_probe.log 2>&1; cat gpurun_out/dsmem_probe.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_i.log 2>&1; tail -1 gpurun_out/gpu_tests_i.log
timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" > gpurun_out/ab26i.log 2>&1
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 2 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" > gpurun_out/ab22i.log 2>&1
timeout 900 python tools/ab_env.py --scale 28 --steps 2 --repeat 1 --variants "ETB_BASE=1" "ETB_L2_PERSIST=1" > gpurun_out/ab28i.log 2>&1
cat gpurun_out/ab26i.log gpurun_out/ab22i.log gpurun_out/ab28i.log
