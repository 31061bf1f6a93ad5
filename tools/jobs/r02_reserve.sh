mkdir -p gpurun_out
for r in 2 0 8 16 32; do
  BCMG_RESERVE_SMS=$r timeout 600 python tools/config_probe.py --config 5 --n 65536 --tiles 128,256,1024 --dtypes f32 --reps 2 | sed "s/^{/{\"reserve\": $r, /" >> gpurun_out/reserve.jsonl 2>> gpurun_out/reserve.err
done
