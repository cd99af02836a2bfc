mkdir -p gpurun_out/r3w
timeout 1500 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_X=0" "ETB_SPLIT_TDW=12" "ETB_SPLIT_TDW=20" "ETB_SPLIT_TDW=16 ETB_SPLIT_RATIO=1.7" "ETB_X=1" > gpurun_out/r3w/ab26.log 2>&1
