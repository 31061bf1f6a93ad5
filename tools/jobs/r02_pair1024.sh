mkdir -p gpurun_out
: > gpurun_out/pair1024.jsonl
for round in 1 2; do
for V in 2 3; do
  BCMG_PAIR_PANELS=$V timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 1024 --reps 2 2>>gpurun_out/pair1024.err | sed "s/^{/{\"pp\": $V, \"round\": $round, /" >> gpurun_out/pair1024.jsonl
done
done
