mkdir -p gpurun_out
timeout 1500 python tools/ab_env.py --scale 26 --repeat 2 --variants "ETB_REPLAY_TAG=r4" "ETB_LIB=tools/variants/r6/libetbfs_b200.so" "ETB_LIB=tools/variants/r8/libetbfs_b200.so" > gpurun_out/r2o_ab26.log 2>&1
timeout 900 python tools/ab_env.py --scale 22 --repeat 2 --variants "ETB_REPLAY_TAG=r4" "ETB_LIB=tools/variants/r8/libetbfs_b200.so" > gpurun_out/r2o_ab22.log 2>&1
timeout 900 python tools/sanitize_run.py > gpurun_out/r2o_san_plain.log 2>&1 && timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/r2o_racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2o_racecheck.log
