timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_mp_plumbing.py -x -q > gpurun_out/t_ii.log 2>&1; tail -1 gpurun_out/t_ii.log
for G in 2 8; do
timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --parts $G --variants "ETB_BASE=1" > gpurun_out/ab26ii_$G.log 2>&1
done
timeout 600 python tools/ab_env.py --scale 22 --steps 3 --repeat 1 --parts 8 --variants "ETB_BASE=1" > gpurun_out/ab22ii_8.log 2>&1
cat gpurun_out/ab26ii_*.log gpurun_out/ab22ii_8.log
