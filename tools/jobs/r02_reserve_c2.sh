mkdir -p gpurun_out
: > gpurun_out/reserve_c2.jsonl
for R in 2 8 16 24 32; do
  BCMG_RESERVE_SMS=$R timeout 300 python tools/kernel_split.py --dtype f64 --n 32768 --t 1024 | sed "s/^{/{\"reserve\": $R, /" >> gpurun_out/reserve_c2.jsonl 2>&1
done
for R in 2 8 16; do
  BCMG_RESERVE_SMS=$R timeout 300 python tools/kernel_split.py --dtype f32 --n 65536 --t 1024 | sed "s/^{/{\"reserve\": $R, /" >> gpurun_out/reserve_c2.jsonl 2>&1
done
