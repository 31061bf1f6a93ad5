mkdir -p gpurun_out
timeout 1500 python tools/config_probe.py --config 5 --d 8 --reps 2 > gpurun_out/c5_last.jsonl 2> gpurun_out/c5_last.err
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo rc=$? >> gpurun_out/smoke_last.log
timeout 1200 python bench.py > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err; echo rc=$? >> gpurun_out/bench_last.err
