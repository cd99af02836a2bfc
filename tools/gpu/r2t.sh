mkdir -p gpurun_out
timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/r2t_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:et_bfs_part_kernel -s 2 -c 1 -o gpurun_out/r02_et_bfs_part2_s26_root0 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/r2t_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2t_ncu.log
