mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_cb.log 2>&1; echo rc=$? >> gpurun_out/gpu_cb.log
timeout 300 python tools/timeline.py --dtype f32 --n 65536 --t 1024 --d 8 > gpurun_out/tl_f32_cb.json 2>> gpurun_out/tl_cb.err
timeout 300 python tools/timeline.py --dtype f64 --n 32768 --t 1024 > gpurun_out/tl_c2_cb.json 2>> gpurun_out/tl_cb.err
timeout 1500 python tools/config_probe.py --config 5 --d 8 --reps 2 > gpurun_out/c5_sweep3.jsonl 2> gpurun_out/c5_sweep3.err
