mkdir -p gpurun_out/r3o
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3o/smoke.log 2>&1; echo rc=$? >> gpurun_out/r3o/smoke.log
timeout 1200 python bench.py > gpurun_out/r3o/bench.json 2> gpurun_out/r3o/bench.err; echo rc=$? >> gpurun_out/r3o/bench.err
echo done > gpurun_out/r3o/done.txt
