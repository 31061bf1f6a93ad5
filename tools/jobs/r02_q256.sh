mkdir -p gpurun_out
timeout -k 5 600 python tools/ab_check.py BCMG_TCK_PAIR_EPI 3 4 > gpurun_out/q256_ab.log 2>&1; echo rc=$? >> gpurun_out/q256_ab.log
: > gpurun_out/q256.jsonl
for round in 1 2; do
for U in 3 4; do
  BCMG_TCK_PAIR_EPI=$U timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 256,512 --dtypes f32 --reps 2 2>>gpurun_out/q256.err | sed "s/^{/{\"pe\": $U, \"round\": $round, /" >> gpurun_out/q256.jsonl
done
done
