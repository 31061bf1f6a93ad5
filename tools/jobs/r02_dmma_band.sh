# band order for the DMMA trailing update: bits (GPU suite), speed and DRAM traffic per band width
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/gpu_band.log 2>&1; echo rc=$? >> gpurun_out/gpu_band.log
for b in 0 4 2 8; do BCMG_DMMA_BAND=$b python tools/trail_ab.py --n 131072 --reps 1 | sed "s/^{/{\"band\": $b, /" >> gpurun_out/dmma_band.jsonl; done
for b in 0 4; do BCMG_DMMA_BAND=$b timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:trail_tma --launch-skip 21 --launch-count 1 --csv python tools/trail_traffic.py --n 131072 > gpurun_out/dmma_band_traffic_$b.csv 2>/dev/null; done
