mkdir -p gpurun_out
timeout 1500 python tools/config_probe.py --config 5 --d 8 --reps 2 > gpurun_out/c5_end.jsonl 2> gpurun_out/c5_end.err
timeout 900 python tools/config_probe.py --config 4 --d 8 --reps 1 > gpurun_out/c4_end.jsonl 2> gpurun_out/c4_end.err
timeout 600 python tools/kernel_split.py --dtype f64 --n 32768 --t 1024 > gpurun_out/c2_end.jsonl 2>&1
