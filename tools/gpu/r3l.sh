mkdir -p gpurun_out/r3l
timeout 2400 python tools/ab_env.py --scale 26 --repeat 1 --variants "ETB_SPLIT_RATIO=2.0" "ETB_SPLIT_RATIO=1.0" "ETB_SPLIT_RATIO=3.0" "ETB_SPLIT_RATIO=2.0 ETB_SPLIT_DIV=512" "ETB_SPLIT_RATIO=2.0 ETB_SPLIT_DIV=2048" "ETB_SPLIT_RATIO=0.5" "ETB_SPLIT_RATIO=2.0 ETB_TD_AS_BU=8" > gpurun_out/r3l/ab26.log 2>&1
timeout 2400 python tools/ab_env.py --scale 28 --repeat 1 --variants "ETB_SPLIT_RATIO=0" "ETB_SPLIT_RATIO=2.0" "ETB_SPLIT_RATIO=2.0 ETB_SPLIT_DIV=4096" "ETB_SPLIT_RATIO=1.0" > gpurun_out/r3l/ab28.log 2>&1
