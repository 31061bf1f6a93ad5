mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_subst.log 2>&1; echo rc=$? >> gpurun_out/gpu_subst.log
timeout 1500 python tools/config_probe.py --config 5 --d 8 --reps 2 > gpurun_out/c5_sweep2.jsonl 2> gpurun_out/c5_sweep2.err
