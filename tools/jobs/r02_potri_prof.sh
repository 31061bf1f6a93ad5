mkdir -p gpurun_out
timeout 900 python tools/profile_kernels.py --routine potri --dtype c128 --n 65536 --t 512 --d 8 --top 30 > gpurun_out/potri_prof.json 2> gpurun_out/potri_prof.err
