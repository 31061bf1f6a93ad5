mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -x --timeout 300 -k "potri or loopback or bit_exact or config4" > gpurun_out/gpu_wacc.log 2>&1; echo rc=$? >> gpurun_out/gpu_wacc.log
timeout 900 python tools/config_probe.py --config 4 --d 8 --reps 1 > gpurun_out/c4_wacc.jsonl 2> gpurun_out/c4_wacc.err
timeout 900 python tools/config_probe.py --config 4 --d 1 --reps 1 >> gpurun_out/c4_wacc.jsonl 2>> gpurun_out/c4_wacc.err
timeout 900 python tools/profile_kernels.py --routine potri --dtype c128 --n 65536 --t 512 --d 8 --top 12 > gpurun_out/potri_prof_wacc.json 2> gpurun_out/potri_prof_wacc.err
