mkdir -p gpurun_out
timeout -k 5 900 python tools/ab_check.py BCMG_TCK_PAIR_EPI 1 2 > gpurun_out/pairepi2_check.log 2>&1; echo rc=$? >> gpurun_out/pairepi2_check.log
for U in 1 2; do
  BCMG_TCK_PAIR_EPI=$U timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 256,512,1024,2048 --reps 1 > gpurun_out/pairepi2_$U.jsonl 2> gpurun_out/pairepi2_$U.err
done
