timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/t_aa.log 2>&1; tail -1 gpurun_out/t_aa.log
for G in 2 8; do
timeout 1200 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --parts $G --variants "ETB_BASE=1" "ETB_LIB=tools/variants/parthead/libetbfs_b200.so" > gpurun_out/ab26aa_$G.log 2>&1
done
cat gpurun_out/ab26aa_*.log
