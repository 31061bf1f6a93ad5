mkdir -p gpurun_out
: > gpurun_out/reserve2.jsonl
for R in 2 8 16 24; do
  BCMG_RESERVE_SMS=$R timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 256,512,1024,2048 --reps 2 2>>gpurun_out/reserve2.err | sed "s/^{/{\"reserve\": $R, /" >> gpurun_out/reserve2.jsonl
done
