V="ETB_BASE=1 ETB_TD_AS_BU=3 ETB_TD_AS_BU=5 ETB_LIB=tools/variants/lf32/libetbfs_b200.so ETB_LIB=tools/variants/lf128/libetbfs_b200.so ETB_LIB=tools/variants/sw15/libetbfs_b200.so ETB_LIB=tools/variants/sw3/libetbfs_b200.so"
timeout 2400 python tools/ab_env.py --scale 26 --steps 3 --repeat 2 --variants $V > gpurun_out/ab26bb.log 2>&1
timeout 1200 python tools/ab_env.py --scale 22 --steps 3 --repeat 1 --variants ETB_BASE=1 ETB_TD_AS_BU=3 ETB_TD_AS_BU=5 ETB_LIB=tools/variants/lf32/libetbfs_b200.so ETB_LIB=tools/variants/lf128/libetbfs_b200.so > gpurun_out/ab22bb.log 2>&1
cat gpurun_out/ab26bb.log gpurun_out/ab22bb.log
