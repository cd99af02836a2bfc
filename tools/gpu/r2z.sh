mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 22 --repeat 2 --variants "ETB_SMALL_MODE3=1e30" "ETB_SMALL_MODE3=2000000" "ETB_SMALL_MODE3=500000" "ETB_SMALL_MODE3=2000000 ETB_TD_AS_BU=2" > gpurun_out/r2z_ab22.log 2>&1
timeout 900 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_SMALL_MODE3=1e30" > gpurun_out/r2z_ab26.log 2>&1
