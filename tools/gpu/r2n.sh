mkdir -p gpurun_out
nproc > gpurun_out/r2n_env.txt; free -g >> gpurun_out/r2n_env.txt
s=$SECONDS; timeout 1800 python bench.py > gpurun_out/r2n_bench.log 2> gpurun_out/r2n_bench.err; echo rc=$? wall=$((SECONDS-s)) >> gpurun_out/r2n_bench.log
s=$SECONDS; timeout 1800 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2n_ref.log 2> gpurun_out/r2n_ref.err; echo rc=$? wall=$((SECONDS-s)) >> gpurun_out/r2n_ref.log
