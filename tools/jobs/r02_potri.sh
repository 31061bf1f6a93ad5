# grouped potri product GEMM: potri parity tests, then config 4 at 8 and 1 logical devices
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "potri or config4 or reservation or invert or loopback" > gpurun_out/gpu_potri.log 2>&1; echo rc=$? >> gpurun_out/gpu_potri.log
timeout 900 python tools/config_probe.py --config 4 --n 65536 --d 8 --reps 1 > gpurun_out/config4_d8.jsonl 2> gpurun_out/config4_d8.err
timeout 900 python tools/config_probe.py --config 4 --n 65536 --d 1 --reps 1 > gpurun_out/config4_d1.jsonl 2> gpurun_out/config4_d1.err
