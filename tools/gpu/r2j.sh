mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_TD_AS_BU=3" "ETB_TD_AS_BU=4" "ETB_TD_AS_BU=5" "ETB_TD_AS_BU=6" > gpurun_out/r2j_ab26.log 2>&1
ETB_TD_AS_BU=4 timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "not s26" > gpurun_out/r2j_parity.log 2>&1; echo rc=$? >> gpurun_out/r2j_parity.log
