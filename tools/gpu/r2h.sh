mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_HOT_WORDS=0" "ETB_HOT_WORDS=4096" "ETB_HOT_WORDS=16384" "ETB_HOT_WORDS=47000" "ETB_HOT_WORDS=16384 ETB_HOT_MIN=1000000" > gpurun_out/r2h_ab26.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --repeat 2 --variants "ETB_HOT_WORDS=0" "ETB_HOT_WORDS=4096 ETB_HOT_MIN=100000" "ETB_HOT_WORDS=47000 ETB_HOT_MIN=100000" > gpurun_out/r2h_ab22.log 2>&1
