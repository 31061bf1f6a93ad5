mkdir -p gpurun_out
: > gpurun_out/reserve3.jsonl
for round in 1 2; do
for R in 2 8 12; do
  BCMG_RESERVE_SMS=$R timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 2048 --reps 2 2>>gpurun_out/reserve3.err | sed "s/^{/{\"reserve\": $R, \"round\": $round, /" >> gpurun_out/reserve3.jsonl
done
done
