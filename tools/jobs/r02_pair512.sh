mkdir -p gpurun_out
: > gpurun_out/pair512.jsonl
for round in 1 2; do
for V in 1 2; do
  BCMG_PAIR_PANELS=$V timeout 900 python tools/config_probe.py --config 5 --d 8 --tiles 512 --reps 2 2>>gpurun_out/pair512.err | sed "s/^{/{\"pp\": $V, \"round\": $round, /" >> gpurun_out/pair512.jsonl
done
done
BCMG_PAIR_PANELS=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x > gpurun_out/pair512_tests.log 2>&1; echo rc=$? >> gpurun_out/pair512_tests.log
