mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode > gpurun_out/r2e_bench.log 2>&1; echo rc=$? >> gpurun_out/r2e_bench.log
timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/r2e_plain26.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/prof_s26 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/r2e_ncu26.log 2>&1; echo rc=$? >> gpurun_out/r2e_ncu26.log
timeout 900 python tools/traffic_capture.py --scale 28 --roots 16 > gpurun_out/r2e_plain28.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:et_bfs_kernel --csv --log-file gpurun_out/traffic_s28.csv python tools/traffic_capture.py --scale 28 --roots 16 > gpurun_out/r2e_ncu28.log 2>&1; echo rc=$? >> gpurun_out/r2e_ncu28.log
