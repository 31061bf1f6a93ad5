mkdir -p gpurun_out
timeout -k 5 900 python tools/ab_check.py BCMG_TCK_UNIT2 0 1 > gpurun_out/unit2_check.log 2>&1; echo rc=$? >> gpurun_out/unit2_check.log
for U in 0 1; do
  BCMG_TCK_UNIT2=$U timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 > gpurun_out/unit2_f32_$U.jsonl 2>&1
  BCMG_TCK_UNIT2=$U timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 > gpurun_out/unit2_c64_$U.jsonl 2>&1
done
if grep -q "rc=0" gpurun_out/unit2_check.log; then
  timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_unit2.log 2>&1; echo rc=$? >> gpurun_out/gpu_unit2.log
fi
