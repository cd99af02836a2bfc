mkdir -p gpurun_out/s28
timeout 600 python tools/s28_reference_check.py --scale 20 --roots 0 1 > gpurun_out/s28/check_s20.log 2>&1; echo rc=$? >> gpurun_out/s28/check_s20.log
tail -3 gpurun_out/s28/check_s20.log
( while true; do free -g | awk 'NR==2{print $3}' >> gpurun_out/s28/mem.log; sleep 10; done ) &
MP=$!
timeout 3000 python tools/s28_reference_check.py --scale 28 --roots 0 1 2 3 > gpurun_out/s28/check_s28.log 2>&1; echo rc=$? >> gpurun_out/s28/check_s28.log
kill $MP
cat gpurun_out/s28/check_s28.log; sort -n gpurun_out/s28/mem.log | tail -1
