mkdir -p gpurun_out
timeout -k 5 900 python tools/ab_check.py BCMG_TCK_PAIR_EPI 0 1 > gpurun_out/pairepi_check.log 2>&1; echo rc=$? >> gpurun_out/pairepi_check.log
if grep -q "rc=0" gpurun_out/pairepi_check.log; then
for U in 0 1; do
  BCMG_TCK_PAIR_EPI=$U timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 > gpurun_out/pairepi_f32_$U.jsonl 2>&1
  BCMG_TCK_PAIR_EPI=$U timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 > gpurun_out/pairepi_c64_$U.jsonl 2>&1
done
BCMG_TCK_PAIR_EPI=1 timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k potrs > gpurun_out/pairepi_loop.log 2>&1; echo rc=$? >> gpurun_out/pairepi_loop.log
fi
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_pairepi.log 2>&1; echo rc=$? >> gpurun_out/gpu_pairepi.log
