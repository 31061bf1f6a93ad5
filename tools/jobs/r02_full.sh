mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_full.log 2>&1; echo rc=$? >> gpurun_out/gpu_full.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo rc=$? >> gpurun_out/smoke_full.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$? >> gpurun_out/bench_full.err
