mkdir -p gpurun_out
s=$SECONDS; timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2v_gpu_tests.log 2>&1; echo rc=$? wall=$((SECONDS-s)) >> gpurun_out/r2v_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2v_smoke.log
