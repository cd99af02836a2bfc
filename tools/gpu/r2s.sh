mkdir -p gpurun_out
timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/r2s_plain26.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/r02_et_bfs_s26_root0 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/r2s_ncu26.log 2>&1
timeout 600 python tools/one_root.py --scale 26 --index 2 --reps 3 > gpurun_out/r2s_plain26b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/r02_et_bfs_s26_slowroot python tools/one_root.py --scale 26 --index 2 --reps 3 > gpurun_out/r2s_ncu26b.log 2>&1
timeout 600 python tools/one_root.py --scale 22 --index 0 --reps 3 > gpurun_out/r2s_plain22.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/r02_et_bfs_s22_root0 python tools/one_root.py --scale 22 --index 0 --reps 3 > gpurun_out/r2s_ncu22.log 2>&1
for sc in 22 26 28; do
timeout 900 python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/r2s_tplain$sc.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:et_bfs_kernel --csv --log-file gpurun_out/r02_traffic_s$sc.csv python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/r2s_tncu$sc.log 2>&1
done
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode --emulate-partitions "" > gpurun_out/r2s_benchplain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_s26.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary 0 --no-paper-mode --emulate-partitions "" > gpurun_out/r2s_launches.log 2>&1
echo done > gpurun_out/r2s_done.txt
