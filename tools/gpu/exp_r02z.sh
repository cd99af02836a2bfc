timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/or_p2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:et_bfs_part_kernel -s 2 -c 1 -o gpurun_out/part2_s26_root0 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/ncu_p2.log 2>&1; echo rc=$? >> gpurun_out/ncu_p2.log
