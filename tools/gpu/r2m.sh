mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity_full.py -x -q -k s26 > gpurun_out/r2m_parity26.log 2>&1; echo rc=$? >> gpurun_out/r2m_parity26.log
timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/r2m_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:et_bfs_part_kernel -s 2 -c 1 -o gpurun_out/prof_s26_part2 python tools/one_root.py --scale 26 --index 0 --reps 3 --parts 2 > gpurun_out/r2m_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2m_ncu.log
