timeout 600 python tools/root_profile.py --scale 22 --roots 8 --cold > gpurun_out/rp22.log 2>&1
timeout 600 python tools/block_balance.py --scale 22 --index 0 1 > gpurun_out/bb22.log 2>&1
