mkdir -p gpurun_out
timeout 1500 python tools/config_probe.py --config 5 --d 8 --reps 2 > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.err
