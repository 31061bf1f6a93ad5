mkdir -p gpurun_out
for spec in "21 1" "20 4"; do set -- $spec
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:trail_tma --launch-skip $1 --launch-count $2 --csv python tools/trail_traffic.py --n 131072 > gpurun_out/trail_traffic_s$1_c$2.csv 2>/dev/null
done
