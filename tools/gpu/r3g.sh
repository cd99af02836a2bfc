mkdir -p gpurun_out/r3g
timeout 900 python tools/block_balance.py --scale 26 --index 0 27 58 28 6 > gpurun_out/r3g/bb26.log 2>&1
