for t in 1.5 2 4 8 0; do
ETB_TD_AS_BU=$t timeout 600 python tools/root_profile.py --scale 26 --roots 64 > gpurun_out/rp26_tdbu_$t.log 2>&1
done
