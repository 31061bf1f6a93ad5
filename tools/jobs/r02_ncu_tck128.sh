mkdir -p gpurun_out /tmp/ncu
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tck_trail --launch-skip 20 --launch-count 1 -o /tmp/ncu/tck_t128_pair python tools/config_probe.py --config 5 --n 65536 --tiles 128 --dtypes f32 --reps 1 > gpurun_out/tck_t128_pair.log 2>&1; echo rc=$? >> gpurun_out/tck_t128_pair.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tck_trail --launch-skip 7 --launch-count 1 -o /tmp/ncu/tck_t1024_umma2 python tools/config_probe.py --config 5 --n 65536 --tiles 1024 --dtypes f32 --reps 1 > gpurun_out/tck_t1024_umma2.log 2>&1; echo rc=$? >> gpurun_out/tck_t1024_umma2.log
for r in tck_t128_pair tck_t1024_umma2; do
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>&1
done
ls -la gpurun_out/
