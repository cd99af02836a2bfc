mkdir -p gpurun_out
timeout 900 python tools/root_profile.py --scale 22 --roots 12 --cold > gpurun_out/r2y_rp22.log 2>&1
ETB_TD_AS_BU=0 timeout 900 python tools/root_profile.py --scale 22 --roots 12 --cold > gpurun_out/r2y_rp22_notdbu.log 2>&1
timeout 900 python tools/root_profile.py --scale 26 --roots 12 --cold > gpurun_out/r2y_rp26.log 2>&1
