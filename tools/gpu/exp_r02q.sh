timeout 600 python tools/block_balance.py --scale 26 --index 0 2 5 > gpurun_out/bb26.log 2>&1
cat gpurun_out/bb26.log
