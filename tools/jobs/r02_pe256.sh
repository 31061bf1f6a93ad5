mkdir -p gpurun_out
: > gpurun_out/pe256.jsonl
for round in 1 2; do
for U in 1 2; do
  BCMG_TCK_PAIR_EPI=$U timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 256,512 --dtypes c64 --reps 2 2>>gpurun_out/pe256.err | sed "s/^{/{\"pe\": $U, \"round\": $round, /" >> gpurun_out/pe256.jsonl
done
done
