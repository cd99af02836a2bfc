mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo rc=$? >> gpurun_out/final/bench.err
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary "" --no-paper-mode --emulate-partitions "" > gpurun_out/final/benchplain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_s26.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --secondary "" --no-paper-mode --emulate-partitions "" > gpurun_out/final/launches.log 2>&1
for sc in 22 26 28; do
timeout 900 python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/final/tplain$sc.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:et_bfs_kernel --csv --log-file gpurun_out/final/traffic_s$sc.csv python tools/traffic_capture.py --scale $sc --roots 16 > gpurun_out/final/tncu$sc.log 2>&1
done
timeout 600 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/final/plain_s26_root0.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:et_bfs_kernel -s 2 -c 1 -o gpurun_out/final/et_bfs_s26_root0 python tools/one_root.py --scale 26 --index 0 --reps 3 > gpurun_out/final/ncu_s26_root0.log 2>&1
echo done > gpurun_out/final/done.txt
