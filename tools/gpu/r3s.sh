mkdir -p gpurun_out/r3s
timeout 1200 python bench.py > gpurun_out/r3s/bench.json 2> gpurun_out/r3s/bench.err; echo rc=$? >> gpurun_out/r3s/bench.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3s/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r3s/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3s/smoke.log 2>&1; echo rc=$? >> gpurun_out/r3s/smoke.log
