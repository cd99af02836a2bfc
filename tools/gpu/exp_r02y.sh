timeout 600 python tools/root_profile.py --scale 26 --roots 8 --cold > gpurun_out/rp26_p1.log 2>&1
timeout 600 python tools/root_profile.py --scale 26 --roots 8 --cold --parts 2 > gpurun_out/rp26_p2.log 2>&1
timeout 600 python tools/part_balance.py --scale 26 --parts 2 --roots 3 > gpurun_out/pb26.log 2>&1
