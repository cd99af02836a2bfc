mkdir -p gpurun_out/r3t
for sc in 26 28; do
timeout 900 python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/r3t/tplain$sc.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:et_bfs_kernel --csv --log-file gpurun_out/r3t/traffic_s$sc.csv python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/r3t/tncu$sc.log 2>&1
done
for spec in "26 27 s26_splitroot" "26 0 s26_root0"; do
  set -- $spec
  timeout 600 python tools/one_root.py --scale $1 --index $2 --reps 3 > gpurun_out/r3t/plain_$3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/r3t/et_bfs_$3 python tools/one_root.py --scale $1 --index $2 --reps 3 > gpurun_out/r3t/ncu_$3.log 2>&1
done
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary "" --no-paper-mode --emulate-partitions "" > gpurun_out/r3t/benchplain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r3t/launches_s26.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary "" --no-paper-mode --emulate-partitions "" > gpurun_out/r3t/launches.log 2>&1
timeout 900 python tools/root_profile.py --cold --scale 26 > gpurun_out/r3t/rp26.log 2>&1
echo done > gpurun_out/r3t/done.txt
