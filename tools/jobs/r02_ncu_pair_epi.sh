mkdir -p gpurun_out /tmp/ncu
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:tck_trail_kernelILi256ELi6E --launch-skip 6 --launch-count 1 -o /tmp/ncu/tck_t128_pairepi python tools/config_probe.py --config 5 --d 8 --n 65536 --tiles 128 --dtypes f32 --reps 1 > gpurun_out/tck_t128_pairepi.log 2>&1; echo rc=$? >> gpurun_out/tck_t128_pairepi.log
ncu -i /tmp/ncu/tck_t128_pairepi.ncu-rep --page raw --csv > gpurun_out/tck_t128_pairepi.raw.csv 2>&1
ncu -i /tmp/ncu/tck_t128_pairepi.ncu-rep --page details --csv > gpurun_out/tck_t128_pairepi.details.csv 2>&1
