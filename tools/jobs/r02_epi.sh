mkdir -p gpurun_out
timeout -k 5 600 python tools/ab_check.py BCMG_TCK_EPI 0 1 > gpurun_out/epi_check.log 2>&1; echo rc=$? >> gpurun_out/epi_check.log
if grep -q "rc=0" gpurun_out/epi_check.log; then
  timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_epi.log 2>&1; echo rc=$? >> gpurun_out/gpu_epi.log
  for e in 0 1; do BCMG_TCK_EPI=$e timeout 600 python tools/config_probe.py --config 5 --n 65536 --tiles 128 --dtypes f32,c64 --reps 2 > gpurun_out/epi_$e.jsonl 2>gpurun_out/epi_$e.err; done
fi
