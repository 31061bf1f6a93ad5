mkdir -p gpurun_out /tmp/ncu
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tck_trail --launch-skip 21 --launch-count 3 -o /tmp/ncu/tck_t128_epi python tools/config_probe.py --config 5 --n 65536 --tiles 128 --dtypes f32 --reps 1 > gpurun_out/tck_t128_epi.log 2>&1; echo rc=$? >> gpurun_out/tck_t128_epi.log
ncu -i /tmp/ncu/tck_t128_epi.ncu-rep --page details --csv > gpurun_out/tck_t128_epi.details.csv 2>&1
ncu -i /tmp/ncu/tck_t128_epi.ncu-rep --page raw --csv > gpurun_out/tck_t128_epi.raw.csv 2>&1
ncu -i /tmp/ncu/tck_t128_epi.ncu-rep --page source --csv > gpurun_out/tck_t128_epi.source.csv 2>&1
ls -la gpurun_out/
