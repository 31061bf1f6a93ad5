mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_nativeb.log 2>&1; echo rc=$? >> gpurun_out/gpu_nativeb.log
for V in 1 0; do
  BCMG_CPLX_NATIVE_B=$V timeout 600 python tools/config_probe.py --config 4 --d 8 > gpurun_out/c4_nativeb_d8_$V.jsonl 2> gpurun_out/c4_nativeb_d8_$V.err
done
timeout 600 python tools/config_probe.py --config 4 --d 1 > gpurun_out/c4_nativeb_d1_1.jsonl 2> gpurun_out/c4_nativeb_d1_1.err
timeout 900 python tools/profile_kernels.py --routine potri --dtype c128 --n 65536 --t 512 --d 8 --top 30 > gpurun_out/potri_prof_nb.json 2> gpurun_out/potri_prof_nb.err
