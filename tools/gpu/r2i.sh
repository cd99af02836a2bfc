mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_TD_AS_BU=0" "ETB_TD_AS_BU=1" "ETB_TD_AS_BU=2" "ETB_TD_AS_BU=4" "ETB_TD_AS_BU=8" > gpurun_out/r2i_ab26.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --repeat 2 --variants "ETB_TD_AS_BU=0" "ETB_TD_AS_BU=1" "ETB_TD_AS_BU=2" "ETB_TD_AS_BU=4" > gpurun_out/r2i_ab22.log 2>&1
