mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo rc=$? >> gpurun_out/bench_r02.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:trail_tma --launch-skip 20 --launch-count 4 --csv python tools/trail_traffic.py --n 131072 > gpurun_out/trail_traffic_n131072.csv 2> gpurun_out/trail_traffic.err; echo rc=$? >> gpurun_out/trail_traffic.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tck_trail --launch-skip 40 --launch-count 1 -o gpurun_out/tck_t128_n65536 python tools/config_probe.py --config 5 --n 65536 --tiles 128 --dtypes f32 --reps 1 > gpurun_out/tck_ncu.log 2>&1; echo rc=$? >> gpurun_out/tck_ncu.log
