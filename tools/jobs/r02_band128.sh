mkdir -p gpurun_out
for B in 8 16 32 64; do
  BCMG_TRAIL_BAND=$B timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 128 > gpurun_out/band_f32_$B.jsonl 2>&1
  BCMG_TRAIL_BAND=$B BCMG_TCK_EPI=1 timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 > gpurun_out/band_c64_$B.jsonl 2>&1
  BCMG_TRAIL_BAND=$B BCMG_TCK_EPI=0 timeout 600 python tools/kernel_split.py --dtype c64 --n 65536 --t 128 > gpurun_out/band_c64e0_$B.jsonl 2>&1
  BCMG_TRAIL_BAND=$B timeout 600 python tools/kernel_split.py --dtype f32 --n 65536 --t 256 > gpurun_out/band_f32t256_$B.jsonl 2>&1
done
