mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_q.log 2>&1; echo rc=$? >> gpurun_out/gpu_q.log
timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 128 --reps 2 > gpurun_out/c5_q.jsonl 2> gpurun_out/c5_q.err
timeout 600 python tools/stress.py --cases 60 --seed 41 --dtypes f32 --tiles 128 --nmax 4000 --dcheck 1 > gpurun_out/stress7.jsonl 2> gpurun_out/stress7.err
