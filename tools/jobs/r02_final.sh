mkdir -p gpurun_out
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; echo rc=$? >> gpurun_out/smoke_r02.log
timeout 1200 python bench.py > gpurun_out/bench_r02_final.json 2> gpurun_out/bench_r02_final.err; echo rc=$? >> gpurun_out/bench_r02_final.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err; echo rc=$? >> gpurun_out/bench_r02_reference.err
